#!/bin/bash
# bench.py smoke of every mode: N=1 default, C3/C5 single, gloo 2-rank one-device.
out=gpurun_out/${1:-r2b}; mkdir -p $out
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --config C3 --steps 100 --no-cpu-baseline --no-c5 > $out/bench_C3.json 2> $out/bench_C3.err
timeout 600 python bench.py --config C5 --steps 50 --no-cpu-baseline --no-c5 > $out/bench_C5.json 2> $out/bench_C5.err
BQG_BENCH_BACKEND=gloo BQG_BENCH_ONE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --no-comparators --c5-steps 3 \
  > $out/bench_gloo2.json 2> $out/bench_gloo2.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err
ls -la $out
