#!/bin/bash
# round-2 check A: GPU tests, reference suite via the shim, calibration study,
# bench, and the axis-0 FIR A/B launch list
cd "$(dirname "$0")/.."
O=gpurun_out
python -m pytest tests -m gpu -x -q -k "not parity3d_full" > $O/r2a_gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> $O/r2a_gpu_tests.log
tools/run_reference_suite.sh run -x -q > $O/r2a_refsuite.log 2>&1; echo "refsuite rc=$?" >> $O/r2a_refsuite.log
tools/run_reference_suite.sh run -q > $O/r2a_refsuite_all.log 2>&1; echo "refsuite rc=$?" >> $O/r2a_refsuite_all.log
timeout 600 python tools/calib_study.py 3,4,5 > $O/r2a_calib.jsonl 2> $O/r2a_calib.err
python tools/prof_cfg2.py --batch 32 --iters 1 > $O/r2a_prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/r2a_launch_persist.csv python tools/prof_cfg2.py --batch 32 --iters 1 > /dev/null 2>&1
MR_AX0_CLASSIC=1 python tools/prof_cfg2.py --batch 32 --iters 1 > $O/r2a_prof_plain2.log 2>&1 && \
MR_AX0_CLASSIC=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/r2a_launch_classic.csv python tools/prof_cfg2.py --batch 32 --iters 1 > /dev/null 2>&1
python -m pytest tests/test_parity3d_full_gpu.py -x -q -s > $O/r2a_full3d.log 2>&1; echo "full3d rc=$?" >> $O/r2a_full3d.log
