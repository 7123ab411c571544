#!/bin/bash
# A/B switches of the cfg2 bench: MR_VEL_CLASSIC=1 (round-1 velocity kernels)
cd "$(dirname "$0")/.."
run() { python bench.py --no-cpu-baseline --e2e-steps 1 $2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', 'ms/step', round(d['ms_per_step'],3), {k:round(v*1e3,1) for k,v in d['kernels_ms'].items()})"; }
run default
MR_VEL_CLASSIC=1 run classic_velocity
run groups1 "--groups 1"
run groups4 "--groups 4"
