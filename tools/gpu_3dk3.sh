set -x
O=gpurun_out/k3d3
mkdir -p $O
timeout 600 python -m pytest tests/test_parity3d_gpu.py -x -q > $O/tests3d.log 2>&1; echo "3d tests $?"; tail -n1 $O/tests3d.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"
for c in 4 3 5; do timeout 600 python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; echo "cfg$c exit $?"; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
ncu --metrics $M --clock-control none -k "regex:k_.*3d|k_fir|k_smooth" -c 1200 --csv --log-file $O/launches_cfg4b4.csv python tools/prof_cfg2.py --config 4 --batch 4 --iters 1 > $O/ncu_cfg4.log 2>&1; echo "ncu cfg4 $?"
