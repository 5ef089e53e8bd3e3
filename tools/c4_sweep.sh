# C4 batch sweep (BASELINE configs[3]): b = 1 is the grouped step (128 calls),
# b >= 2 single calls; one JSON summary per b.
for b in 1 2 4 8 16 32 64 128 256; do
  timeout 300 python bench.py --config C4 --batch $b --steps 20 --warmup 5 --no-cpu-baseline --no-comparators --no-sweep --no-c5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'b': $b, 'us_per_call': round(d['us_per_call'],2), 'latency_us': d.get('latency',{}).get('us_per_call'), 'e2e_us': round(d['e2e']['us_per_call'],2) if 'e2e' in d else None, 'key_gbs': d['value'], 'lds_frac': d['roofline'].get('lds_frac'), 'rel': d['parity_rel_fro']}))"
done
