#!/bin/bash
cd "$(dirname "$0")/.."
run() { python bench.py --no-cpu-baseline --e2e-steps 1 $2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', 'ms/step', round(d['ms_per_step'],3), {k:round(v*1e3,1) for k,v in d['kernels_ms'].items()})"; }
run default
MR_AX0_CLASSIC=1 run ax0_classic
MR_FIR_SMEM_PAD=32768 run pad32k
MR_FIR_SMEM_PAD=65536 run pad64k
MR_FIR_SMEM_PAD=32768 run pad32k_g4 "--groups 4"
MR_FIR_SMEM_PAD=65536 run pad64k_g4 "--groups 4"
MR_FIR_SMEM_PAD=65536 run pad64k_g3 "--groups 3"
