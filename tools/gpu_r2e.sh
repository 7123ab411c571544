#!/bin/bash
# round-2 check E: new tests (canary, batched line search), whole reference suite incl. CLI / IO / acceptance
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
python -m pytest tests/test_canary_gpu.py tests/test_optimize_batch_gpu.py -m gpu -q -x > $O/r2e_new_tests.log 2>&1; echo "new tests rc=$?" >> $O/r2e_new_tests.log
tail -15 $O/r2e_new_tests.log
tools/run_reference_suite.sh run -q -rf -x > $O/r2e_refsuite.log 2>&1; echo "refsuite rc=$?" >> $O/r2e_refsuite.log
tail -30 $O/r2e_refsuite.log
