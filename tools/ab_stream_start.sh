#!/bin/bash
# A/B of the key-stream start (BQG_DEBUG_FLAGS bit 21 = 2097152): stream form
# (C4 single call; C2 group of one with the latency form skipped, bit 14) --
# bit 21 restores the all-at-once ring fill.  (The C2/C1 lines measured a
# latency-form variant where bit 21 made key piece 0 land alone first: 5.52
# -> 5.6 us, worse, removed -- bit 21 is a no-op there now.)
out=${1:-gpurun_out/ab_stream_start.txt}; mkdir -p $(dirname $out); : > $out
for rep in 1 2; do
 for f in 0 2097152; do echo "flag=$f $(BQG_DEBUG_FLAGS=$f timeout 300 python tools/chain_time.py C4 1 50 | tail -1)" >> $out; done
 for f in 16384 2113536; do echo "flag=$f $(BQG_DEBUG_FLAGS=$f timeout 300 python tools/chain_time.py C2 1 50 | tail -1)" >> $out; done
 for c in C2 C1; do for f in 0 2097152; do echo "flag=$f $(BQG_DEBUG_FLAGS=$f timeout 300 python tools/chain_time.py $c 1 50 | tail -1)" >> $out; done; done
done
cat $out
