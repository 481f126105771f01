#!/bin/bash
# bounds-checked build (device asserts) over the sanitizer workload and the GPU parity suite
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
OCTAX_CHECKED=1 timeout 600 python scripts/sanitize_run.py > gpurun_out/checked_run.log 2>&1; echo "checked workload rc=$?"
tail -2 gpurun_out/checked_run.log
OCTAX_CHECKED=1 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/checked_pytest.log 2>&1; echo "checked pytest rc=$?"
tail -2 gpurun_out/checked_pytest.log
