timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/timeline.py C2 40 | grep -vE "slowest|^[0-9]"
timeout 300 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('us/call', round(d['us_per_call'],3), 'GB/s', d['value'], 'e2e us', round(d['e2e']['us_per_call'],2))"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_kernel.py --config C2 --calls 6 > /dev/null 2>&1; grep -E "biqgemm_fast|finalize" gpurun_out/launches_c2.csv | tail -4 | cut -d, -f5,14-
