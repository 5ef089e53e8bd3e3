#!/bin/bash
# Round-2 late evidence (final round-2 code: ring starts, latency layout and any-NB clusters, grouped-form crossover): GPU tests, bench lines (default C2, the reference
# arm, C1, C4, C3, C5), the mu sweep of the fast / exact paths.
out=gpurun_out/final_r2g; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $out/smi.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu > $out/gpu_tests.txt 2>&1
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err
for c in C1 C4; do timeout 600 python bench.py --config $c --no-comparators --no-c5 > $out/bench_$c.json 2> $out/bench_$c.err; done
for c in C3 C5; do timeout 900 python bench.py --config $c --steps 50 --no-c5 > $out/bench_$c.json 2> $out/bench_$c.err; done
timeout 600 python tools/exact_speed.py > $out/mu_speed.txt 2>&1
ls -la $out
