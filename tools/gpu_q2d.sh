#!/bin/bash
# quick 2D iteration: velocity / veladj operator parity + goldens, then the cfg2 bench (A/B via env)
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
python -m pytest tests/test_parity_gpu.py -m gpu -q -x > $O/q2d_tests.log 2>&1; echo "rc=$?" >> $O/q2d_tests.log
tail -4 $O/q2d_tests.log
python bench.py --no-cpu-baseline > $O/q2d_bench.json 2> $O/q2d_bench.err || tail -5 $O/q2d_bench.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/q2d_bench.json").read().strip().splitlines()[-1])
print("ms/step", d["ms_per_step"], "kernels", d["kernels_ms"], "e2e", d["e2e"]["ms_per_step"])
PY
