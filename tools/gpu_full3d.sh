#!/bin/bash
# slow full-size 3D oracle parity (cfg3 full, cfg4 x 2, cfg5 prefix / 128^3 / mu = 0)
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
MR_FULL_PARITY=1 python -m pytest tests/test_parity3d_full_gpu.py -q -s > $O/full3d_final.log 2>&1; echo "full3d rc=$?" >> $O/full3d_final.log; grep -E "passed|failed|rc=|worst" $O/full3d_final.log
