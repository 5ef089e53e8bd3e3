#!/bin/bash
# Single dependent calls of mid-size m: the latency form (default where its
# shared memory fits) vs the stream form's group of one (BQG_DEBUG_FLAGS=16384
# skips the latency form).  tools/grouped_bench.py's single-call PDL chain.
out=${1:-gpurun_out/ab_single_form.txt}; mkdir -p $(dirname $out); : > $out
for rep in 1 2; do for shape in "4096 4096 3" "6144 4096 3" "8192 4096 3" "8192 4096 1" "11008 4096 2" "8192 2048 4"; do for f in 0 16384; do
  echo "flags=$f m,n,beta=$shape $(BQG_DEBUG_FLAGS=$f timeout 120 python tools/grouped_bench.py C2 1 $shape 2>&1 | grep 'single-call')" >> $out
done; done; done
cat $out
