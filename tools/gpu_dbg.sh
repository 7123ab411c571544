#!/bin/bash
cd "$(dirname "$0")/.."
for args in "1 16 16 3" "2 64 128 24" "2 98 152 12" "1 20 24 24" "3 512 512 24" "2 130 200 9" "2 60 36 32" "1 2 4 1" "40 256 256 5"; do echo "== $args"; timeout 120 python tools/dbg_fast2d.py $args 2>&1 | grep -v ok | tail -3; done
timeout 120 python tools/fir_bench.py
