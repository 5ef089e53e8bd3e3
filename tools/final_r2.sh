#!/bin/bash
# Round-2 evidence: GPU tests, bench lines (default C2, reference arm, every config), the C4 batch sweep.
out=gpurun_out/final_r2; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $out/smi.txt 2>&1
python bench.py > $out/bench.json 2> $out/bench.err
python bench.py --impl reference --steps 5 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err
for c in C1 C4; do timeout 600 python bench.py --config $c --no-comparators --no-c5 > $out/bench_$c.json 2> $out/bench_$c.err; done
for c in C3 C5; do timeout 900 python bench.py --config $c --steps 50 --no-c5 > $out/bench_$c.json 2> $out/bench_$c.err; done
bash tools/c4_sweep.sh > $out/c4_sweep.txt 2>&1
ls -la $out
