#!/bin/bash
# A/B of the cluster form's ring start (form 2: b <= 4, 8 <= NB <= 16, MT <= 256):
# default: stage 0 lands alone before the rest is requested; BQG_DEBUG_FLAGS bit 21
# (2097152) = the old all-at-once fill (the run below had the meaning inverted:
# flag=2097152 was the stage-0-first variant).
out=${1:-gpurun_out/ab_cluster_start.txt}; mkdir -p $(dirname $out); : > $out
for rep in 1 2; do for b in 2 3 4; do for f in 0 2097152; do
  echo "flag=$f $(BQG_DEBUG_FLAGS=$f timeout 300 python tools/chain_time.py C2 $b 50 | tail -1)" >> $out
done; done; done
cat $out
