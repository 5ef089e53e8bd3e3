#!/bin/bash
# A/B the grouped form across library variants: tools/ab_variants.sh OUT CFG "v1 v2 ..." ("" = default build)
out=$1; cfg=$2; shift 2
mkdir -p $(dirname $out)
for v in $@; do
  if [ "$v" = "default" ]; then vv=""; else vv=$v; fi
  echo "== variant $v" >> $out
  BQG_LIB_VARIANT=$vv timeout 200 python tools/grouped_bench.py $cfg 128 2>&1 | grep -E "grouped|Error|error" >> $out
done
