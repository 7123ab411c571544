mkdir -p gpurun_out/prof
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/gpu_tests2d.log 2>&1; echo "tests exit $?"; tail -3 gpurun_out/gpu_tests2d.log
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "cfg2 exit $?"
ncu --metrics gpu__time_duration.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 100 --csv --log-file gpurun_out/prof/launches_cfg2_split.csv python tools/prof_cfg2.py --iters 1 > gpurun_out/prof/l.log 2>&1; echo "ncu $?"
