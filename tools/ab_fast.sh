out=gpurun_out/ab_fast.txt; : > $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_grouped.py -q -x 2>&1 | tail -2 >> $out
bash tools/ab_single.sh gpurun_out/ab_fast_single.txt "oldfast default" "C3 C4:2 C4:4 C4:16 C4:256 C5"
cat $out gpurun_out/ab_fast_single.txt
