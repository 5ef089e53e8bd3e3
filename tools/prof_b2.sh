#!/bin/bash
out=gpurun_out/prof_b2; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_grouped.py -q -x -k shared_workspace > $out/test.txt 2>&1
F="--set full --clock-control none --import-source on"
for b in 2 4; do
timeout 900 ncu $F -k regex:"biqgemm_fast_kernel|finalize_kernel" -s 4 -c 2 -o $out/fast_C4b$b python bench.py --config C4 --batch $b --profile --steps 4 --warmup 3 > $out/fast_C4b$b.log 2>&1
done
ls -la $out; cat $out/test.txt | tail -2
