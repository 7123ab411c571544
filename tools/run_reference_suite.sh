#!/bin/bash
# Run the reference package's own tests against the B200 facade through the
# `morphreg` shim (tools/morphreg_shim, float64 mode).
#
#   here (container with /root/reference):  tools/run_reference_suite.sh stage
#       copies /root/reference/pkg/tests into baseline/_ref/pkg_tests (git-ignored,
#       travels to the GPU box with the gpurun snapshot; nothing is committed)
#   on the GPU box:                          tools/run_reference_suite.sh run [pytest args]
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
DST="$ROOT/baseline/_ref/pkg_tests"
case "${1:-run}" in
  stage)
    mkdir -p "$DST"
    cp /root/reference/pkg/tests/*.py "$DST/"
    echo "staged $(ls "$DST" | wc -l) files in $DST"
    ;;
  run)
    shift || true
    cd "$DST"
    PYTHONPATH="$ROOT/tools/morphreg_shim:$ROOT" python -m pytest -p no:cacheprovider -q \
      -o addopts="" --rootdir "$DST" \
      test_fields.py test_kernel.py test_integrator.py test_objective.py test_optimizer.py \
      test_synthetic.py test_io_cli.py test_acceptance.py "$@"
    ;;
esac
