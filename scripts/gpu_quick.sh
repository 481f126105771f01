#!/bin/bash
# quick iteration: build, GPU parity tests, bench (headline only unless FULL=1)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q --maxfail=5 -p no:cacheprovider -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
if [ "${FULL:-0}" = "1" ]; then BARGS="--steps 20 --warmup 5"; else BARGS="--steps 20 --warmup 5 --no-e2e --no-cpu"; fi
timeout 600 python bench.py $BARGS > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
python - <<'PY'
import json
try:
    d = json.load(open("gpurun_out/bench.json"))
    print("value %.4g steps/s  ms/step %.3f  bound %s frac %.3f  clocks %s" % (d["value"], d["ms_per_step"], d["roofline"]["bound"], d["roofline"]["frac"], d["clocks"]))
    for s in d.get("sweep", []): print("  sweep", s)
except Exception as e:
    print("bench parse failed", e); print(open("gpurun_out/bench.err").read()[-2000:])
PY
