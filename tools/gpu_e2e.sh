#!/bin/bash
cd "$(dirname "$0")/.."
for c in 4 "8,16,20,20" "4,12,16,16,16" "8,24,32" "16,24,24" "12,16,18,18"; do python bench.py --no-cpu-baseline --e2e-chunks $c 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('chunks','$c','device ms',round(d['ms_per_step'],3),'e2e ms',round(d['e2e']['ms_per_step'],3))"; done
