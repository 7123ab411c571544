set -x
O=gpurun_out/cost3d
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests exit $?"; tail -n1 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"
for c in 4 3 5 2; do timeout 600 python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; echo "cfg$c exit $?"; done
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:cost_terms" -c 4 --csv --log-file $O/launches_cost3d.csv python tools/prof_cfg2.py --config 4 --batch 4 --iters 1 > $O/ncu.log 2>&1; echo "ncu $?"
