#!/bin/bash
# tools/gap_variants.sh OUT CFG v1 v2 ... : launch_gap.py per library variant ("default" = the main build)
out=$1; cfg=$2; shift 2
for v in $@; do
  if [ "$v" = "default" ]; then vv=""; else vv=$v; fi
  echo "== variant $v" >> $out
  BQG_LIB_VARIANT=$vv timeout 200 python tools/launch_gap.py $cfg 2>&1 | grep -E "launches=  1|launches= 16|rror" >> $out
done
