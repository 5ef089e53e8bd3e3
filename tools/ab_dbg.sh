#!/bin/bash
# tools/ab_dbg.sh OUT CFG "dbg values" : grouped bench (group 128) under BQG_TEX_DBG flags
out=$1; cfg=$2; shift 2
for v in $@; do
  echo "== dbg $v variant ${BQG_LIB_VARIANT:-default}" >> $out
  BQG_TEX_DBG=$v timeout 200 python tools/grouped_bench.py $cfg 128 2>&1 | grep -E "group  128|Error|error" >> $out
done
