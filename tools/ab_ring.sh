#!/bin/bash
# A/B of the two-kernel form's key-ring start: ring depth cap (BQG_FAST_RMAX)
# and the old all-at-once ring fill (BQG_DEBUG_FLAGS bit 21 = 2097152; the
# default lands stage 0 alone first).  50 PDL-chained calls per config.
out=${1:-gpurun_out/ab_ring.txt}; mkdir -p $(dirname $out); : > $out
for rep in 1 2; do
for c in "C4 2" "C4 4" "C3 0" "C4 16" "C4 64" "C5 0"; do set -- $c
  for v in "6 2097152" "6 0" "2 0" "4 0"; do set -- $c $v
    r=$(BQG_FAST_RMAX=$3 BQG_DEBUG_FLAGS=$4 timeout 300 python tools/chain_time.py $1 $2 50 2>&1 | tail -1)
    echo "rmax=$3 flags=$4 $r" >> $out
  done
done; done
cat $out
