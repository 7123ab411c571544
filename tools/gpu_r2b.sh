#!/bin/bash
# round-2 check B: full GPU suite (incl. full-size 3D parity), reference suite,
# benches (default, deterministic, cfg5 mu=0)
cd "$(dirname "$0")/.."
O=gpurun_out
python -m pytest tests -m gpu -q -k "not parity3d_full" > $O/r2b_gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> $O/r2b_gpu_tests.log
tools/run_reference_suite.sh run -q -rf > $O/r2b_refsuite.log 2>&1; echo "refsuite rc=$?" >> $O/r2b_refsuite.log
python bench.py > $O/r2b_bench.json 2> $O/r2b_bench.err
python bench.py --deterministic --no-cpu-baseline > $O/r2b_bench_det.json 2>> $O/r2b_bench.err
python bench.py --config 5 --mu 0 --steps 3 --no-cpu-baseline > $O/r2b_bench_cfg5mu0.json 2>> $O/r2b_bench.err
python -m pytest tests/test_parity3d_full_gpu.py -q -s > $O/r2b_full3d.log 2>&1; echo "full3d rc=$?" >> $O/r2b_full3d.log
