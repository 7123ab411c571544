set -x
O=gpurun_out/s6
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests exit $?"
tail -3 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"; tail -2 $O/smoke.log
for c in 2 1 3 4 5; do timeout 600 python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; echo "cfg$c exit $?"; done
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref exit $?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_cfg2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_cfg2.log 2>&1; echo "ncu cfg2 $?"
M=gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active
ncu --metrics $M --clock-control none -c 200 --csv --log-file $O/launches_cfg4b4.csv python tools/prof_cfg2.py --config 4 --batch 4 --iters 1 > $O/ncu_cfg4.log 2>&1; echo "ncu cfg4 $?"
