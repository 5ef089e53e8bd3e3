python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -3 gpurun_out/bench2.err; cat gpurun_out/bench2.json
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_kernel.py --config C2 --calls 6 > /dev/null 2>&1; grep biqgemm_fast gpurun_out/launches_c2.csv | grep duration | tail -4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:biqgemm_fast -s 2 -c 1 -o gpurun_out/prof_c2b python tools/prof_kernel.py --config C2 --calls 4 > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
