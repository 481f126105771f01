#!/bin/bash
# full evidence pass: gpu tests, smoke, default bench (JSON line), ncu launch list of the same
# command, ncu --set full of one headline step launch
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -2 gpurun_out/smoke.log
CMD="python bench.py"
timeout 900 $CMD > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 $CMD > gpurun_out/bench_plain2.json 2> gpurun_out/bench_plain2.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
ENVS=1048576 TAG=prof_full bash scripts/gpu_ncu.sh
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print("value %.4g ms/step %.3f frac %.3f e2e %.3g cpu %.3g cores %s clocks %s" % (d["value"], d["ms_per_step"], d["roofline"]["frac"], d["e2e"]["value"], d["cpu_baseline"]["value"], d["cpu_baseline"]["cores"], d["clocks"]))
for s in d["sweep"]: print("  ", s)
PY
