#!/bin/bash
# FIR microbench (+ optional ncu of kernels matching $1, report name $2)
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
python tools/fir_bench.py ${FIR_ARGS:-} 2>&1 | tee $O/fir_bench.txt
MR_VEL_CLASSIC=1 MR_VADJ_CLASSIC=1 python tools/fir_bench.py 2>&1 | sed 's/^/classic /' | tee -a $O/fir_bench.txt
if [ -n "$1" ]; then
  python tools/fir_bench.py --iters 2 --sets 2 > $O/fir_plain.log 2>&1 &&
  ncu --set full --import-source on --clock-control none -k "regex:$1" -s 4 -c ${3:-2} -f -o $O/$2 python tools/fir_bench.py --iters 2 --sets 2 > $O/ncu_$2.log 2>&1
  echo "ncu rc=$?"
fi
