#!/bin/bash
# Round-2 evidence pass: full GPU tests, bench lines, ncu of the texture kernel.
out=gpurun_out/ev_r2; mkdir -p $out
timeout 1800 python -m pytest tests -q -m gpu > $out/gpu_tests.txt 2>&1
python bench.py > $out/bench.json 2> $out/bench.err
F="--set full --clock-control none --import-source on"
timeout 900 ncu $F -k regex:biqgemm_tex_kernel -s 3 -c 1 -o $out/full_tex_C2 python bench.py --profile --steps 4 --warmup 3 > $out/full_tex_C2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -c 600 --log-file $out/launches_C2.csv python bench.py --steps 20 --warmup 5 --no-comparators --no-cpu-baseline --no-sweep --no-c5 > $out/launches_C2.log 2>&1
ls -la $out; tail -3 $out/gpu_tests.txt
