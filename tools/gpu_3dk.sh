set -x
O=gpurun_out/k3d
mkdir -p $O
timeout 600 python -m pytest tests/test_parity3d_gpu.py -x -q > $O/tests3d.log 2>&1; echo "3d tests $?"; tail -1 $O/tests3d.log
for K in 1 2 4; do MR_3D_K=$K timeout 600 python bench.py --config 4 --no-cpu-baseline > $O/bench_cfg4_k$K.json 2> $O/bench_cfg4_k$K.err; echo "cfg4 K=$K $?"; done
MR_3D_K=2 timeout 600 python bench.py --config 3 --no-cpu-baseline > $O/bench_cfg3_k2.json 2> $O/bench_cfg3_k2.err; echo "cfg3 $?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
for K in 1 2 4; do MR_3D_K=$K ncu --metrics $M --clock-control none -c 2500 --csv --log-file $O/launches_cfg4b4_k$K.csv python tools/prof_cfg2.py --config 4 --batch 4 --iters 1 > $O/ncu_k$K.log 2>&1; echo "ncu K=$K $?"; done
