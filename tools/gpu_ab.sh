#!/bin/bash
cd "$(dirname "$0")/.."
run() { python bench.py --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', 'ms/step', round(d['ms_per_step'],3), {k:round(v*1e3,1) for k,v in d['kernels_ms'].items()})"; }
run new_all
MR_VADJ_CLASSIC=1 run new_vel_classic_adj
MR_VEL_CLASSIC=1 run classic_vel_new_adj
MR_VEL_CLASSIC=1 MR_VADJ_CLASSIC=1 run classic_all
