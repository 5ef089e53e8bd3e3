#!/bin/bash
# A/B library variants on single-call configs: tools/ab_single.sh OUT "v1 v2" "CFG[:b] ..."
out=$1; vars=$2; cfgs=$3
mkdir -p $(dirname $out)
for rep in 1 2; do
for c in $cfgs; do
for v in $vars; do
  if [ "$v" = "default" ]; then vv=""; else vv=$v; fi
  cfg=${c%%:*}; b=${c#*:}; [ "$b" = "$c" ] && b=0
  r=$(BQG_LIB_VARIANT=$vv timeout 300 python bench.py --config $cfg --batch $b --steps 50 --warmup 5 --no-comparators --no-cpu-baseline --no-c5 --no-sweep 2>&1 | tail -1)
  python - "$v $c" "$r" >> $out <<'PY'
import json,sys
v,r=sys.argv[1],sys.argv[2]
try:
    d=json.loads(r); print(f"{v:18s} us/call {d['us_per_call']:.3f} sustained {d['sustained']['us_per_call']:.3f} lds_frac {d['roofline'].get('lds_frac')} sm {d['clocks']['sm_mhz']} rel {d['parity_rel_fro']:.2e}")
except Exception as e:
    print(v, "ERR", r[:300])
PY
done; done; done
cat $out
