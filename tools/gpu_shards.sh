#!/bin/bash
# per-rank step time of a W-rank cfg2 job, measured as rank 0's shard on one GPU
cd "$(dirname "$0")/.."
for wg in "8 2" "8 4" "8 8" "4 2" "4 4" "4 8"; do set -- $wg; python bench.py --no-cpu-baseline --e2e-steps 1 --shard-of $1 --groups $2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ranks',$1,'groups',$2,'pairs on this rank',64//$1,'ms/step',round(d['ms_per_step'],3))"; done
