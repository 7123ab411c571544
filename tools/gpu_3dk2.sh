set -x
O=gpurun_out/k3d2
mkdir -p $O
timeout 600 python -m pytest tests/test_parity3d_gpu.py -x -q > $O/tests3d.log 2>&1; echo "3d tests $?"; tail -1 $O/tests3d.log
MR_3D_KA=1 MR_3D_KE=1 timeout 600 python -m pytest tests/test_parity3d_gpu.py -x -q > $O/tests3d_k1.log 2>&1; echo "3d tests k1 $?"; tail -1 $O/tests3d_k1.log
timeout 600 python bench.py --config 4 --no-cpu-baseline > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "cfg4 $?"
MR_3D_KA=1 timeout 600 python bench.py --config 4 --no-cpu-baseline > $O/bench_cfg4_ka1.json 2> $O/bench_cfg4_ka1.err; echo "cfg4 ka1 $?"
MR_3D_KE=4 timeout 600 python bench.py --config 4 --no-cpu-baseline > $O/bench_cfg4_ke4.json 2> $O/bench_cfg4_ke4.err; echo "cfg4 ke4 $?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
for KA in 1 2 4; do MR_3D_KA=$KA MR_3D_KE=$KA ncu --metrics $M --clock-control none -k "regex:adjoint3d|divseed|epi3d|product3d" -c 400 --csv --log-file $O/launches_cfg4b4_ka$KA.csv python tools/prof_cfg2.py --config 4 --batch 4 --iters 1 > $O/ncu_ka$KA.log 2>&1; echo "ncu KA=$KA $?"; done
