timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in C2 C3 C5; do timeout 600 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c us/call', round(d['us_per_call'],2), 'GB/s', d['value'])"; done
BQG_DEBUG_FLAGS=128 timeout 600 python bench.py --config C3 --steps 300 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3 2-kernel us/call', round(d['us_per_call'],2))"
