#!/bin/bash
# Single dependent calls with NB not a power of 2 (clusters of 3-12 CTAs): the
# latency form (default) vs the stream form's group of one (BQG_DEBUG_FLAGS=16384).
out=${1:-gpurun_out/ab_single_form2.txt}; mkdir -p $(dirname $out); : > $out
for rep in 1 2; do for shape in "4096 3072 3" "3072 3072 3" "8192 3072 2" "2048 1536 2" "3000 2400 1" "4096 1280 4"; do for f in 0 16384; do
  echo "flags=$f m,n,beta=$shape $(BQG_DEBUG_FLAGS=$f timeout 120 python tools/grouped_bench.py C2 1 $shape 2>&1 | grep 'single-call')" >> $out
done; done; done
cat $out
