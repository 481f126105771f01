#!/bin/bash
# build the in-tree library, run the GPU parity suite against it, then A/B-time ab/*.so
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
[ -z "$SKIP_TESTS" ] && timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
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
