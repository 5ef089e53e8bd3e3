#!/bin/bash
# Late round-2 evidence: C4 batch sweep after the ring-start change, ncu launch
# lists (C4 b=2, C5) and full captures of the two-kernel gather kernel (C4 b=2,
# C5) and the latency kernel (C2, sized shared memory).
out=gpurun_out/prof_r2e; mkdir -p $out
bash tools/c4_sweep.sh > $out/c4_sweep.txt 2>&1
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
timeout 600 ncu $M --log-file $out/launches_C4b2.csv python bench.py --config C4 --batch 2 --profile --steps 8 --warmup 3 > $out/launches_C4b2.log 2>&1
timeout 900 ncu $M --log-file $out/launches_C5.csv python bench.py --config C5 --profile --steps 4 --warmup 3 > $out/launches_C5.log 2>&1
F="--set full --clock-control none --import-source on"
timeout 900 ncu $F -k regex:"biqgemm_fast_kernel|finalize_kernel" -s 4 -c 2 -o $out/full_fast_C4b2 python bench.py --config C4 --batch 2 --profile --steps 4 --warmup 3 > $out/full_fast_C4b2.log 2>&1
timeout 900 ncu $F -k regex:"biqgemm_fast_kernel|finalize_kernel" -s 4 -c 2 -o $out/full_fast_C5 python bench.py --config C5 --profile --steps 4 --warmup 3 > $out/full_fast_C5.log 2>&1
timeout 900 ncu $F -k regex:biqgemm_latency_kernel -s 8 -c 1 -o $out/full_lat_C2 python bench.py --profile --steps 4 --warmup 3 > $out/full_lat_C2.log 2>&1
ls -la $out
