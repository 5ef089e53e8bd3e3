#!/bin/bash
out=gpurun_out/r2cols; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_grouped.py tests/test_sharded.py -q -x -m gpu > $out/tests.txt 2>&1
for b in 2 3 4 8; do
  timeout 300 python bench.py --config C4 --batch $b --steps 50 --warmup 5 --no-cpu-baseline --no-comparators --no-sweep --no-c5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4 b=$b', round(d['us_per_call'],2), 'form', d['config'].get('form'), 'lds', d['roofline'].get('lds_frac'), 'rel', d['parity_rel_fro'])" >> $out/res.txt
  timeout 300 python bench.py --config C2 --batch $b --steps 50 --warmup 5 --no-cpu-baseline --no-comparators --no-sweep --no-c5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2 b=$b', round(d['us_per_call'],2), 'form', d['config'].get('form'), 'lds', d['roofline'].get('lds_frac'), 'rel', d['parity_rel_fro'])" >> $out/res.txt
done
for sf in 4 16 64; do
  BQG_TEX_SEPFIN=$sf timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-comparators --no-c5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sepfin $sf', d['group_sweep'], round(d['us_per_call'],3))" >> $out/res.txt
done
tail -3 $out/tests.txt >> $out/res.txt
cat $out/res.txt
