#!/bin/bash
# A/B of programmatic dependent launch (ab/a_cur.so: plain launches, ab/$PDL_SO.so: with PDL):
# the whole GPU suite against the PDL build, then step / fused timing on both kernels
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
OCTAX_LIB=$PWD/ab/${PDL_SO:-b_pdl}.so timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_pdl.log 2>&1; echo "pdl suite rc=$? $(tail -1 gpurun_out/pytest_pdl.log)"
rm -f gpurun_out/ab_pdl.jsonl
for r in 1 2 3; do
  for so in ab/*.so; do
    OCTAX_LIB=$PWD/$so timeout 300 python scripts/kernel_crossover.py --kernels warp --tag $(basename $so .so) \
      --games pong_standin target_shooter_level3 --ns 512 2048 4096 >> gpurun_out/ab_pdl.jsonl 2>/dev/null
    OCTAX_LIB=$PWD/$so timeout 300 python scripts/kernel_crossover.py --kernels lane --tag $(basename $so .so) \
      --games pong_standin target_shooter_level3 --ns ${LANE_NS:-16384 65536 262144 1048576} >> gpurun_out/ab_pdl.jsonl 2>/dev/null
  done
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/ab_pdl.jsonl"):
    r = json.loads(l); d[(r["game"], r["kernel"], r["n"], r["tag"])].append((r["step_steps_per_s"], r["fused_steps_per_s"]))
for k in sorted(d):
    v = d[k]; print(f"{k[0]:22s} {k[1]:5s} {k[2]:8d} {k[3]:8s} step {max(a for a, b in v):.4g} fused {max(b for a, b in v):.4g}")
PY
