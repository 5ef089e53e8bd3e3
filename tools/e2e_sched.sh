out=gpurun_out/e2e_sched.txt; : > $out
for sch in "" "64" "32" "16,48,48,16" "16,32,32,32,16" "8,24,32,32,24,8" "32,64,32" "16,56,56" "24,40,40,24" "8,16,32,48,16,8"; do
  BQG_E2E_SCHEDULE=$sch timeout 300 python tools/e2e_sched.py 40 >> $out 2>&1
done
cat $out
