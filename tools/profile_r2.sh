#!/bin/bash
# Round-2 ncu evidence for profiles/: launch lists of the bench commands
# (cold, serialised; -c bounds the count) and full captures of each hot kernel.
out=gpurun_out/prof_r2; mkdir -p $out
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
timeout 900 ncu $M -c 600 --log-file $out/launches_C2.csv python bench.py --steps 20 --warmup 5 --no-comparators --no-cpu-baseline --no-sweep --no-c5 > $out/launches_C2.log 2>&1
timeout 600 ncu $M --log-file $out/launches_C4.csv python bench.py --config C4 --profile --steps 4 --warmup 3 > $out/launches_C4.log 2>&1
timeout 600 ncu $M --log-file $out/launches_C3.csv python bench.py --config C3 --profile --steps 8 --warmup 3 > $out/launches_C3.log 2>&1
timeout 900 ncu $M --log-file $out/launches_C5.csv python bench.py --config C5 --profile --steps 4 --warmup 3 > $out/launches_C5.log 2>&1
F="--set full --clock-control none --import-source on"
timeout 900 ncu $F -k regex:biqgemm_tex_kernel -s 3 -c 1 -o $out/full_tex_C2 python bench.py --profile --steps 4 --warmup 3 > $out/full_tex_C2.log 2>&1
timeout 900 ncu $F -k regex:biqgemm_tex_kernel -s 3 -c 1 -o $out/full_tex_C4 python bench.py --config C4 --profile --steps 4 --warmup 3 > $out/full_tex_C4.log 2>&1
timeout 900 ncu $F -k regex:biqgemm_latency_kernel -s 8 -c 1 -o $out/full_lat_C2 python bench.py --profile --steps 4 --warmup 3 > $out/full_lat_C2.log 2>&1
timeout 900 ncu $F -k regex:"biqgemm_fast_kernel|finalize_kernel" -s 4 -c 2 -o $out/full_fast_C3 python bench.py --config C3 --profile --steps 4 --warmup 3 > $out/full_fast_C3.log 2>&1
timeout 900 ncu $F -k regex:"biqgemm_fast_kernel|finalize_kernel" -s 4 -c 2 -o $out/full_fast_C5 python bench.py --config C5 --profile --steps 4 --warmup 3 > $out/full_fast_C5.log 2>&1
ls -la $out
