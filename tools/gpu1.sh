set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30
timeout 300 python bench.py --steps 2000 --warmup 50 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -3 gpurun_out/bench1.err; cat gpurun_out/bench1.json
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_kernel.py --config C2 --calls 6 > /dev/null 2>&1; tail -8 gpurun_out/launches_c2.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:biqgemm_fast -s 2 -c 1 -o gpurun_out/prof_c2 python tools/prof_kernel.py --config C2 --calls 4 > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
