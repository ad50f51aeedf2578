#!/bin/bash
# Ship the reference's test files (from /root/reference, present only in the
# build container) to a B200 inside the gpurun command line and run them
# against this package through the maskfold alias. Output:
# gpurun_out/reference_suite.log. Optional "$1": more shell to run after it
# on the same box.
set -eu
B64=$(tar czf - -C /root/reference/pkg --exclude=__pycache__ tests | base64 -w0)
exec /usr/local/graft/bin/gpurun --timeout "${TIMEOUT:-1500}" -- \
  "mkdir -p /tmp/mf_suite && echo $B64 | base64 -d | tar xz -C /tmp/mf_suite && \
   bash tools/run_reference_suite.sh /tmp/mf_suite/tests > gpurun_out/reference_suite.log 2>&1; \
   tail -3 gpurun_out/reference_suite.log; ${1:-true}" | grep -v "^\[gpurun\] sending"
