#!/bin/bash
# tree check after a warp-kernel change: GPU suite, smoke, bench line, warp-kernel crossover sweep
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k boundary > gpurun_out/pytest_boundary.log 2>&1; echo "boundary rc=$? $(tail -1 gpurun_out/pytest_boundary.log)"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_final.log
tail -3 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_final.log
t0=$(date +%s)
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$? wall $(( $(date +%s) - t0 )) s"
cut -c1-300 gpurun_out/bench_final.json
rm -f gpurun_out/hybrid_crossover.jsonl
for r in 1 2; do timeout 300 python scripts/kernel_crossover.py --kernels warp --tag hybrid --games pong_standin brix_standin target_shooter_level1 --ns 512 2048 2049 4096 >> gpurun_out/hybrid_crossover.jsonl 2>/dev/null; done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/hybrid_crossover.jsonl"):
    r = json.loads(l); d[(r["game"], r["n"])].append((r["step_steps_per_s"], r["fused_steps_per_s"]))
for k in sorted(d):
    v = d[k]; print(f"{k[0]:22s} {k[1]:6d} hybrid step {max(a for a, b in v):.4g} fused {max(b for a, b in v):.4g}")
PY
