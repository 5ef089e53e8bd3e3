#!/bin/bash
# End-of-round evidence under gpurun: GPU tests, bench lines (default C2,
# reference arm, every config), the C4 batch sweep, and ncu captures for
# profiles/ (stream + latency kernels for C2/C4, fast form for C3/C5).
#   bash tools/final_round.sh r1
tag=${1:-r1}
out=gpurun_out/final_$tag; mkdir -p $out
python -m pytest tests -x -q -m gpu > $out/gpu_tests.txt 2>&1
python bench.py > $out/bench.json 2> $out/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err
for c in C1 C3 C4 C5; do timeout 600 python bench.py --config $c --steps 200 --warmup 5 > $out/bench_$c.json 2> $out/bench_$c.err; done
bash tools/c4_sweep.sh > $out/c4_sweep.txt 2>&1
bash tools/profile_round.sh $tag C2
bash tools/profile_round.sh $tag C4
for spec in "C3 4096 4096 2 32" "C5 65536 8192 2 8"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"biqgemm_fast_kernel|finalize_kernel" -s 4 -c 2 \
    -o gpurun_out/prof_$tag/fast_$1 python tools/fast_sweep.py $2 $3 $4 $5 4 > gpurun_out/prof_$tag/fast_$1.log 2>&1
done
ls -la $out gpurun_out/prof_$tag
