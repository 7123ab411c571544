set -x
O=gpurun_out/cost2d
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests exit $?"; tail -n1 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"
timeout 600 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "cfg2 exit $?"
timeout 600 python bench.py --config 1 > $O/bench_cfg1.json 2> $O/bench_cfg1.err; echo "cfg1 exit $?"
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:cost_terms" -c 10 --csv --log-file $O/launches_cost.csv python tools/prof_cfg2.py --batch 32 --iters 2 > $O/ncu.log 2>&1; echo "ncu $?"
