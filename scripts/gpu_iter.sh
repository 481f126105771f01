#!/bin/bash
# iteration pass: build, all GPU parity tests, bench with per-game rows (no e2e / cpu)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q --maxfail=5 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print("value %.4g ms/step %.3f bound %s frac %.3f clocks %s" % (d["value"], d["ms_per_step"], d["roofline"]["bound"], d["roofline"]["frac"], d["clocks"]))
for g in d["games"]: print("  %-24s %.4g" % (g["game"], g["steps_per_s"]))
PY
if [ -n "$TAG" ]; then ENVS=1048576 TAG=$TAG bash scripts/gpu_ncu.sh; fi
