python bench.py --steps 3 --warmup 3 --no-gmres --no-cpu-baseline --no-cube > gpurun_out/s4_bench_short.json 2> gpurun_out/s4_bench_short.err && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02c_launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-gmres --no-cpu-baseline --no-cube > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_near_stream|k_far_tree" -s 6 -c 2 -o gpurun_out/r02c_full -f python bench.py --steps 3 --warmup 3 --no-gmres --no-cpu-baseline --no-cube > gpurun_out/ncu2.log 2>&1
ncu -i gpurun_out/r02c_full.ncu-rep --page raw --csv > gpurun_out/r02c_full_raw.csv 2>/dev/null
python tools/step_trace.py cfg2 > gpurun_out/r02c_step_trace.txt 2>&1
PROBE_HIST=1 python tools/overhead_probe.py 2 > gpurun_out/r02c_overhead_probe.txt 2>&1
H2B_NEAR_TRACE= H2B_TREE_TRACE=1 python tools/tree_trace.py cfg2 > gpurun_out/r02c_tree_trace.txt 2>&1
