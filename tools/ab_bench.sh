#!/bin/bash
# A/B library variants through bench.py (sustained, clocks sampled):
#   tools/ab_bench.sh OUT "default v1 v2 ..." [bench args]
out=$1; vars=$2; shift 2
mkdir -p $(dirname $out)
for rep in 1 2; do
for v in $vars; do
  if [ "$v" = "default" ]; then vv=""; else vv=$v; fi
  r=$(BQG_LIB_VARIANT=$vv timeout 300 python bench.py --no-comparators --no-cpu-baseline "$@" 2>&1 | tail -1)
  python - "$v" "$r" >> $out <<'PY'
import json,sys
v,r=sys.argv[1],sys.argv[2]
try:
    d=json.loads(r); print(f"{v:12s} us/call {d['us_per_call']:.4f} frac {d['roofline']['frac']:.4f} lat {d['latency']['us_per_call']:.3f} e2e {d['e2e']['us_per_call']:.3f} sm {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
except Exception as e:
    print(v, "ERR", r[:300])
PY
done
done
cat $out
