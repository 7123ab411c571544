mkdir -p gpurun_out/it
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/it/tests.log 2>&1; echo "tests exit $?"; tail -1 gpurun_out/it/tests.log
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/it/bench_cfg2.json 2> gpurun_out/it/bench_cfg2.err; echo "cfg2 $?"
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/it/bench_cfg4.json 2> gpurun_out/it/bench_cfg4.err; echo "cfg4 $?"
M=gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active
ncu --metrics $M --clock-control none -k "regex:axis0" -c 8 --csv --log-file gpurun_out/it/launches_axis0.csv python tools/prof_cfg2.py --batch 32 --iters 1 > /dev/null 2>&1; echo "ncu $?"
