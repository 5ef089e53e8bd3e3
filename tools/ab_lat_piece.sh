#!/bin/bash
# A/B of the latency form's key-piece size (BQG_LAT_PIECE KiB per TMA copy):
# variants built by tools/build_variant.sh p4/p16/p32; 50 PDL-chained calls.
out=${1:-gpurun_out/ab_lat_piece.txt}; mkdir -p $(dirname $out); : > $out
for rep in 1 2; do for c in C2 C1; do for v in default p4 p16 p32; do
  vv=$v; [ "$v" = "default" ] && vv=""
  echo "piece=$v $(BQG_LIB_VARIANT=$vv timeout 120 python tools/chain_time.py $c 1 50 | tail -1)" >> $out
done; done; done
for beta in 1 4; do for v in default p16 p32; do vv=$v; [ "$v" = "default" ] && vv=""
  echo "piece=$v $(BQG_LIB_VARIANT=$vv timeout 120 python tools/lat_chain.py 4096 4096 $beta 200 | tail -1)" >> $out; done; done
cat $out
