#!/bin/bash
# round-2 check C: GPU suite at HEAD, bench A/B (column-first vs classic velocity), FFMA issue-rate probe
cd "$(dirname "$0")/.."
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -q -x -k "not parity3d_full" > $O/r2c_gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> $O/r2c_gpu_tests.log
python bench.py --no-cpu-baseline > $O/r2c_bench.json 2> $O/r2c_bench.err
MR_VEL_CLASSIC=1 python bench.py --no-cpu-baseline > $O/r2c_bench_classic.json 2>> $O/r2c_bench.err
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma_rates tools/probes/ffma_rates.cu && /tmp/ffma_rates > $O/r2c_ffma_rates.txt 2>&1
tail -3 $O/r2c_gpu_tests.log; cat $O/r2c_ffma_rates.txt
