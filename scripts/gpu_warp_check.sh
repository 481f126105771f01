#!/bin/bash
# warp-per-env kernel: the GPU suite with every handle forced onto it, then the lane / warp
# crossover across batch sizes
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
OCTAX_KERNEL=warp timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} \
  > gpurun_out/pytest_gpu_warp.log 2>&1; echo "pytest(warp) rc=$?" >> gpurun_out/pytest_gpu_warp.log
grep -E "passed|failed|rc=" gpurun_out/pytest_gpu_warp.log | tail -3
grep -E "^FAILED" gpurun_out/pytest_gpu_warp.log | head -30
if [ -z "$SKIP_PROBE" ]; then
timeout 900 python scripts/kernel_crossover.py ${PROBE_ARGS} > gpurun_out/kernel_crossover.jsonl 2> gpurun_out/kernel_crossover.err; echo "probe rc=$?"
tail -3 gpurun_out/kernel_crossover.err
fi
