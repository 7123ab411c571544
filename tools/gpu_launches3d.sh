#!/bin/bash
# launch list (ncu gpu__time_duration, cold / serialised) of one grad() at cfg4 with 4 pairs of 128^3
cd "$(dirname "$0")/.."
O=gpurun_out/prof3d_r2; mkdir -p $O
python tools/prof_cfg2.py --config 4 --batch 4 --iters 1 > $O/plain.log 2>&1 || { tail -3 $O/plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_cfg4x4.csv python tools/prof_cfg2.py --config 4 --batch 4 --iters 1 > $O/l.log 2>&1; echo "launches rc=$?"
