#!/bin/bash
# round-2 baseline evidence: ncu --set full (with source) of one headline step launch at 1M
# and at 262,144 envs, for per-line attribution (scripts/ncu_source.py)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
ENVS=1048576 TAG=${TAG1:-r2_full_1M} bash scripts/gpu_ncu.sh
ENVS=262144 TAG=${TAG2:-r2_full_262K} bash scripts/gpu_ncu.sh
ls -la gpurun_out/*.ncu-rep
