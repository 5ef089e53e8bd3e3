#!/bin/bash
# ncu evidence for profiles/: launch list of the bench command (cold, serialised)
# and full captures of the stream kernel and the single-call latency kernel.
# Usage (under gpurun): bash tools/profile_round.sh r1 C2
tag=${1:-r1}; cfg=${2:-C2}
mkdir -p gpurun_out/prof_$tag
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/prof_$tag/launches_$cfg.csv python bench.py --config $cfg --profile --steps 512 --warmup 3 \
  > gpurun_out/prof_$tag/launches_$cfg.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:biqgemm_stream_kernel -s 2 -c 1 \
  -o gpurun_out/prof_$tag/full_$cfg python bench.py --config $cfg --profile --steps 512 --warmup 3 \
  > gpurun_out/prof_$tag/full_$cfg.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:biqgemm_latency_kernel -s 8 -c 1 \
  -o gpurun_out/prof_$tag/lat_$cfg python bench.py --config $cfg --profile --steps 512 --warmup 3 \
  > gpurun_out/prof_$tag/lat_$cfg.log 2>&1
ls -la gpurun_out/prof_$tag
