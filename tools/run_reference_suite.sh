#!/bin/bash
# Run the reference's OWN pytest suite against this package: `import maskfold`
# resolves to paper_2104_12470_b200 through tests/maskfold_alias (its
# `maskfold.reference` oracle is the installed reference's own module).
#   tools/run_reference_suite.sh <dir holding the reference's tests/> [pytest args]
# Build container: tools/run_reference_suite.sh /root/reference/pkg/tests
#   (host-side tests only; the rest need a B200).
# GPU box: tools/gpu_reference_suite.sh ships the test files inside the gpurun
#   command (they are never copied into this repository).
set -u
SRC=${1:?reference tests dir}; shift
REPO=$(cd "$(dirname "$0")/.." && pwd)
WORK=$(mktemp -d)
cp -r "$SRC" "$WORK/tests"
cd "$WORK/tests"
PYTHONDONTWRITEBYTECODE=1 PYTHONPATH="$REPO/tests/maskfold_alias:$REPO" \
  python -m pytest -q -p no:cacheprovider -rfE "$@"
rc=$?
rm -rf "$WORK"
exit $rc
