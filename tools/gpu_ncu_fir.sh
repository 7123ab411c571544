#!/bin/bash
# ncu --set full of FIR kernels matching $1 -> gpurun_out/$2.ncu-rep (fir_bench.py as the driver)
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
python tools/fir_bench.py --iters 2 --sets 2 ${FIR_ARGS:-} > $O/fir_plain.log 2>&1 &&
ncu --set full --import-source on --clock-control none -k "regex:$1" -s ${4:-0} -c ${3:-2} -f -o $O/$2 python tools/fir_bench.py --iters 2 --sets 2 ${FIR_ARGS:-} > $O/ncu_$2.log 2>&1
echo "ncu rc=$?"
