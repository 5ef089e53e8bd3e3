# C4 batch sweep (BASELINE configs[3]): one bench line per b
for b in 1 2 4 8 16 32 64 128 256; do
  timeout 300 python bench.py --config C4 --batch $b --steps 200 --warmup 5 --group 32 --e2e-group 64 --no-cpu-baseline --no-comparators 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'b': $b, 'us_per_call': round(d['us_per_call'],2), 'latency_us': d['latency']['us_per_call'], 'e2e_us': round(d['e2e']['us_per_call'],2), 'key_gbs': d['value'], 'rel': d['parity_rel_fro']}))"
done
