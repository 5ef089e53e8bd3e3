#!/bin/bash
# Round-2 closing evidence: b>=2 lines, the C4 sweep, ncu of the two-kernel form.
out=gpurun_out/final_r2b; mkdir -p $out
for c in C3 C5; do timeout 900 python bench.py --config $c --steps 50 --no-c5 > $out/bench_$c.json 2> $out/bench_$c.err; done
bash tools/c4_sweep.sh > $out/c4_sweep.txt 2>&1
F="--set full --clock-control none --import-source on"
for c in C3 C5; do
timeout 900 ncu $F -k regex:"biqgemm_fast_kernel|finalize_kernel" -s 4 -c 2 -o $out/full_fast_$c python bench.py --config $c --profile --steps 4 --warmup 3 > $out/full_fast_$c.log 2>&1
done
ls -la $out
