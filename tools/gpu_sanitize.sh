#!/bin/bash
# one compute-sanitizer tool per call: tools/gpu_sanitize.sh memcheck|racecheck|synccheck|initcheck
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
T=${1:-memcheck}
timeout 900 python tools/sanitize_cases.py > $O/sanitize_plain.log 2>&1 || { echo "plain run failed"; tail -5 $O/sanitize_plain.log; exit 1; }
timeout 1500 compute-sanitizer --tool $T --error-exitcode 9 python tools/sanitize_cases.py > $O/sanitize_$T.log 2>&1
echo "$T rc=$?"
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|^ok|ops ok" $O/sanitize_$T.log | tail -20
