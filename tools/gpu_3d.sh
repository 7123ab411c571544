mkdir -p gpurun_out/prof3d
timeout 600 python -m pytest tests/test_parity3d_gpu.py -x -q > gpurun_out/gpu_tests3d.log 2>&1; echo "3d tests $?"; tail -1 gpurun_out/gpu_tests3d.log
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "cfg4 $?"
M=gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -c 100 --csv --log-file gpurun_out/prof3d/launches_cfg4b4.csv python tools/prof_cfg2.py --config 4 --batch 4 --iters 1 > /dev/null 2>&1; echo "ncu $?"
ncu --metrics $M --clock-control none -k "regex:k_divseed3d|k_sl_adjoint3d|k_veladj_epi3d|k_cost_terms3d" -c 60 --csv --log-file gpurun_out/prof3d/launches_cfg4b4_adj.csv python tools/prof_cfg2.py --config 4 --batch 4 --iters 1 > /dev/null 2>&1; echo "ncu $?"
