timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/timeline.py C2 40
timeout 300 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('us/call', round(d['us_per_call'],3), 'GB/s', d['value'], 'e2e us', round(d['e2e']['us_per_call'],2))"
