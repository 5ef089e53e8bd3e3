#!/bin/bash
# A/B of the latency form's shared-memory request: sized to the call (>= 116 KiB,
# default) vs the whole 227 KiB (BQG_LAT_SMEM=full); dependent chains of 200 calls.
out=${1:-gpurun_out/lat_ab2.txt}; mkdir -p $(dirname $out); : > $out
for rep in 1 2 3; do for shape in "4096 1" "4096 2" "4096 3" "4096 4" "1024 1" "2048 2"; do set -- $shape; for v in small full; do
  echo "smem=$v $(BQG_LAT_SMEM=$v timeout 300 python tools/lat_chain.py $1 $1 $2 200 2>&1 | tail -1)" >> $out
done; done; done
cat $out
