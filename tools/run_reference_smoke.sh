#!/bin/bash
# Runs the reference's own Python smoke test (proj/tests/python/test_smoke.py), UNMODIFIED,
# against this implementation through the `babplan` alias (compat/babplan).  The reference tree
# does not exist on the GPU box, so the test file travels in the gpurun command line (written to
# /tmp there), never into this repository:
#   /usr/local/graft/bin/gpurun -- "$(tools/run_reference_smoke.sh --remote-cmd)"
# Locally (with /root/reference present and a GPU) it runs the file in place.
set -e
REF=/root/reference/proj/tests/python/test_smoke.py
if [ "$1" = "--remote-cmd" ]; then
  printf 'mkdir -p /tmp/refsmoke && cat > /tmp/refsmoke/test_smoke.py <<'"'"'REFEOF'"'"'\n'
  cat "$REF"
  printf 'REFEOF\ncd $GRAFT_REPO_ROOT && PYTHONPATH=$PWD/compat:$PWD python -m pytest /tmp/refsmoke/test_smoke.py -v -p no:cacheprovider -rs > gpurun_out/reference_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/reference_smoke.log\n'
  exit 0
fi
cd "$(dirname "$0")/.."
PYTHONPATH=$PWD/compat:$PWD python -m pytest "$REF" -v -p no:cacheprovider -rs
