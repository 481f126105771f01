#!/bin/bash
# full evidence pass: gpu tests, smoke, ncu --set full of one headline step launch (its
# instruction counts feed the bench's ALU roofline), default bench (JSON line), ncu launch
# list of the same command, and (PROTOCOL=1) the paper's rollout protocol
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -2 gpurun_out/smoke.log
ENVS=1048576 TAG=prof_full bash scripts/gpu_ncu.sh
python scripts/ncu_summary.py full gpurun_out/prof_full.ncu-rep gpurun_out/step_full_1M.json --envs 1048576 --game pong_standin > /dev/null 2>&1 && \
  cp gpurun_out/step_full_1M.json profiles/latest_step_full.json && echo "instruction counts refreshed"
CMD="python bench.py"
timeout 900 $CMD > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 $CMD > gpurun_out/bench_plain2.json 2> gpurun_out/bench_plain2.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
if [ -n "$PROTOCOL" ]; then
  timeout 1500 python scripts/paper_protocol.py --out gpurun_out/paper_protocol > gpurun_out/protocol.log 2>&1; echo "protocol rc=$?"
fi
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print("value %.4g ms/step %.3f frac %.3f e2e %.3g (link %s) cpu %.3g cores %s clocks %s" % (d["value"], d["ms_per_step"], d["roofline"]["frac"], d["e2e"]["value"], d["e2e"].get("link"), d["cpu_baseline"]["value"], d["cpu_baseline"]["cores"], d["clocks"]))
for s in d["sweep"]: print("  ", s)
PY
