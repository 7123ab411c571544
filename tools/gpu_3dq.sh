#!/bin/bash
# quick 3D check: parity tests + cfg3 / cfg4 bench
cd "$(dirname "$0")/.."
python -m pytest tests/test_parity3d_gpu.py tests/test_determinism_gpu.py -m gpu -q -x 2>&1 | tail -2
for c in 3 4; do python bench.py --config $c --steps 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg$c ms/step',round(d['ms_per_step'],3),'frac',round(d['step_roofline']['frac'],4))"; done
