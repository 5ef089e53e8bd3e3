#!/bin/bash
out=gpurun_out/r2lat; mkdir -p $out
timeout 300 python tools/timeline_latency.py C2 40 > $out/timeline_C2.txt 2>&1
timeout 300 python tools/timeline_latency.py C1 40 > $out/timeline_C1.txt 2>&1
for f in 16 32 64; do for sub in 32 64 128; do
  BQG_E2E_FIRST=$f BQG_E2E_SUB=$sub timeout 300 python bench.py --steps 20 --no-comparators --no-cpu-baseline --no-sweep --no-c5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('first $f sub $sub e2e', round(d['e2e']['us_per_call'],3), 'dev', round(d['us_per_call'],3), 'sus', round(d['sustained']['us_per_call'],3), d['clocks']['sm_mhz'], d['sustained']['clocks']['sm_mhz'])" >> $out/e2e_sweep.txt
done; done
cat $out/*.txt
