#!/bin/bash
# round-2 check F: batched line search timing (cfg2), full-size 3D parity incl. the slow cfg3 test
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
python tools/optimize_batch_timing.py --config 2 --iters 3 > $O/r2f_optimize_batch_cfg2.json 2> $O/r2f_optimize_batch.err; cat $O/r2f_optimize_batch_cfg2.json; tail -2 $O/r2f_optimize_batch.err
python -m pytest tests/test_host_layers.py tests/test_optimize_batch_gpu.py tests/test_canary_gpu.py -q 2>&1 | tail -2
MR_FULL_PARITY=1 python -m pytest tests/test_parity3d_full_gpu.py -q -s > $O/r2f_full3d.log 2>&1; echo "full3d rc=$?" >> $O/r2f_full3d.log; grep -E "passed|failed|rc=|worst" $O/r2f_full3d.log
