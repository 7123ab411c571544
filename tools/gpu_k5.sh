#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
python tools/prof_cfg2.py --batch 32 --iters 1 > $O/plain.log 2>&1 &&
ncu --set full --import-source on --clock-control none -k "regex:k_cost_terms2d" -c 1 -f -o $O/k5 python tools/prof_cfg2.py --batch 32 --iters 1 > $O/k5.log 2>&1; echo "rc=$?"
