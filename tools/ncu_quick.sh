#!/bin/bash
# usage: tools/ncu_quick.sh <kernel-regex> <name>   (run on the GPU box)
ncu --set full --import-source on --clock-control none -k "regex:$1" -s 2 -c ${3:-1} -o "gpurun_out/$2" \
    python tools/prof_cfg2.py --iters 1 ${PROF_ARGS:-} > "gpurun_out/ncu_$2.log" 2>&1
