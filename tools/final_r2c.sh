#!/bin/bash
# Round-2 evidence after the conflict-free x staging: GPU tests, default bench,
# b>=2 lines, the C4 sweep, launch lists + full captures of the two-kernel form.
out=gpurun_out/final_r2c; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $out/smi.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x > $out/gpu_tests.txt 2>&1
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err
for c in C3 C5; do timeout 900 python bench.py --config $c --steps 50 --no-c5 > $out/bench_$c.json 2> $out/bench_$c.err; done
bash tools/c4_sweep.sh > $out/c4_sweep.txt 2>&1
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
for c in C3 C5; do
timeout 900 ncu $M --log-file $out/launches_$c.csv python bench.py --config $c --profile --steps 8 --warmup 3 > $out/launches_$c.log 2>&1
done
F="--set full --clock-control none --import-source on"
for c in C3 C5; do
timeout 900 ncu $F -k regex:"biqgemm_fast_kernel|finalize_kernel" -s 4 -c 2 -o $out/full_fast_$c python bench.py --config $c --profile --steps 4 --warmup 3 > $out/full_fast_$c.log 2>&1
done
ls -la $out
