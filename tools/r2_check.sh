#!/bin/bash
# Round-2 status pass: GPU tests, default bench line, launch list + one full capture of the grouped texture kernel.
out=gpurun_out/r2a; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $out/smi.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" > $out/lscpu.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $out/gpu_tests.txt 2>&1
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --steps 20 --warmup 3 > $out/bench_s20.json 2> $out/bench_s20.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $out/launches_C2.csv python bench.py --config C2 --profile --steps 512 --warmup 3 > $out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:biqgemm_tex_kernel -s 2 -c 1 \
  -o $out/full_tex_C2 python bench.py --config C2 --profile --steps 512 --warmup 3 > $out/full.log 2>&1
ls -la $out
