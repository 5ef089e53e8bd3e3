out=gpurun_out/lat_ab.txt; : > $out
for v in "" kf p2 p4 kfp2; do
  echo "== variant '$v'" >> $out
  BQG_LIB_VARIANT=$v python tools/timeline_latency.py C2 40 2>&1 | grep -E "pdl_wait|lut_built|gathered|y_stored|keys_issued|keys_all" >> $out
  BQG_LIB_VARIANT=$v timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-comparators --no-sweep --no-c5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('latency', d['latency']['us_per_call'])" >> $out
done
cat $out
