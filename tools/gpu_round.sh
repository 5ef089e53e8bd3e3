# Full measurement pass: bench lines, ncu launch list, ncu full capture.
set -x
mkdir -p gpurun_out/r1
python bench.py > gpurun_out/r1/bench_c2.json 2> gpurun_out/r1/bench_c2.err
for c in C1 C3 C4 C5; do timeout 600 python bench.py --config $c --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/r1/bench_$c.json 2> gpurun_out/r1/bench_$c.err; done
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r1/bench_ref.json 2> gpurun_out/r1/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1/ncu_launches_c2.csv python tools/prof_kernel.py --config C2 --calls 6 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:biqgemm -s 3 -c 1 -o gpurun_out/r1/ncu_full_c2 python tools/prof_kernel.py --config C2 --calls 5 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:biqgemm -s 1 -c 1 -o gpurun_out/r1/ncu_full_c3 python tools/prof_kernel.py --config C3 --calls 3 > /dev/null 2>&1
ls -la gpurun_out/r1
