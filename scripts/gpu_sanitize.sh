#!/bin/bash
# one compute-sanitizer tool per call (B200_PROFILING.md); TOOL=memcheck|racecheck|synccheck|initcheck
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
TOOL=${TOOL:-memcheck}
timeout 300 python scripts/sanitize_run.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitize_$TOOL.log 2>&1
echo "rc=$?"
tail -5 gpurun_out/sanitize_$TOOL.log
