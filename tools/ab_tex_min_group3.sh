#!/bin/bash
# Crossover of the grouped forms (the data behind tex_min_group, biqgemm_stream.cu;
# profiles/ab_grouped_crossover_r2e.txt also holds the G = 1..12 runs): TMA-ring stream form (variant tex64,
# -DBQG_TEX_MIN_GROUP=64) vs the texture form (default) at group sizes around
# the crossover, for several layer shapes (m n beta).
out=${1:-gpurun_out/ab_tex_min_group3.txt}; mkdir -p $(dirname $out); : > $out
run() { # shape G
  for v in default tex64; do vv=$v; [ "$v" = "default" ] && vv=""
    echo "$v m,n,beta=$1 G=$2 $(BQG_LIB_VARIANT=$vv timeout 120 python tools/grouped_bench.py C2 $2 $1 2>&1 | grep -E "\(group +$2\)" | tail -1)" >> $out
  done; }
for g in 10 16; do run "4096 4096 3" $g; done
for g in 16 24 32 48; do run "16384 4096 3" $g; done
for g in 8 12 16 24; do run "8192 4096 3" $g; done
for g in 8 12 16; do run "4096 4096 1" $g; done
for g in 8 16 32; do run "16384 4096 1" $g; done
for g in 8 16 32; do run "11008 4096 2" $g; done
cat $out
