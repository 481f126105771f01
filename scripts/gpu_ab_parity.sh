#!/bin/bash
# A/B with a parity gate: every ab/*.so first runs a GPU parity subset against the oracle
# (OCTAX_LIB points the binding at the variant), then all variants are timed interleaved
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
K=${PARITY_K:-"game_parity or fuzz_rom_parity or quirk_parity or edge_rom or hand_vector or rollout_games or stack_frames_obs"}
for so in ab/*.so; do
  OCTAX_LIB=$PWD/$so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rollout.py -m gpu -q -x \
     -p no:cacheprovider -k "$K" > gpurun_out/parity_$(basename $so .so).log 2>&1
  echo "$(basename $so) parity rc=$? $(tail -1 gpurun_out/parity_$(basename $so .so).log)"
done
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
