#!/bin/bash
# round-2 check D: full GPU suite (not the slow full-size 3D parity), reference suite, default bench
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
python -m pytest tests -m gpu -q -k "not parity3d_full" > $O/r2d_gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> $O/r2d_gpu_tests.log
tail -3 $O/r2d_gpu_tests.log
tools/run_reference_suite.sh run -q -rf > $O/r2d_refsuite.log 2>&1; echo "refsuite rc=$?" >> $O/r2d_refsuite.log
tail -2 $O/r2d_refsuite.log
python bench.py > $O/r2d_bench.json 2> $O/r2d_bench.err; tail -c 600 $O/r2d_bench.json
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
