cd "$(dirname "$0")/.."
for g in 1 2 4 8; do MR_VEL_CLASSIC=1 python bench.py --no-cpu-baseline --groups $g --e2e-steps 1 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('groups',$g,'ms/step',d['ms_per_step'])"; done
