#!/bin/bash
# build, full GPU suite (no -x: every failure listed), A/B timing of ab/*.so, default bench line
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
if [ -z "$SKIP_TESTS" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  tail -4 gpurun_out/pytest_gpu.log
fi
if ls ab/*.so > /dev/null 2>&1; then
  bash scripts/ab_bench.sh > /dev/null 2>&1
  python - <<'PY'
import collections
d = collections.defaultdict(list)
for line in open("gpurun_out/ab.log"):
    _, r, so, g, v = line.split()
    d[(g, so)].append(float(v))
for (g, so), v in sorted(d.items()):
    print("%-24s %-16s %s  max %.4g" % (g, so, " ".join("%.4g" % x for x in v), max(v)))
PY
fi
if [ -z "$SKIP_BENCH" ]; then
  timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
  python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
r = d["roofline"]
print("value %.4g ms/step %.4f bound %s frac %.3f fused %s" % (d["value"], d["ms_per_step"], r["bound"], r["frac"],
      d.get("fused") and "%.4g (x%.3f)" % (d["fused"]["steps_per_s"], d["fused"]["vs_step_mode"])))
for s in d["sweep"]: print("  ", {k: (round(v, 4) if isinstance(v, float) and v < 100 else ("%.4g" % v if isinstance(v, float) else v)) for k, v in s.items()})
print("games", [(g["game"], "%.4g" % g["steps_per_s"]) for g in d["games"]])
PY
fi
