#!/bin/bash
# A/B of the warp kernel's idle-loop fast-forward (ab/a_cur.so: OCTAX_WARP_FF=0, ab/b_ff.so: on):
# parity of each variant (warp kernel forced; includes the idle-loop test), then the crossover sweep
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for so in ab/*.so; do
  OCTAX_KERNEL=warp OCTAX_LIB=$PWD/$so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rollout.py tests/test_gpu_kernels.py -m gpu -q -x \
     -p no:cacheprovider -k "game_parity or fuzz_rom or quirk_parity or rollout_games or idle_loop or edge_rom or frame_skip or deferred or config2" > gpurun_out/parity_$(basename $so .so).log 2>&1
  echo "$(basename $so) parity rc=$? $(tail -1 gpurun_out/parity_$(basename $so .so).log)"
done
rm -f gpurun_out/ab_ff.jsonl
for r in $(seq ${ROUNDS:-2}); do
  for so in ab/*.so; do
    OCTAX_LIB=$PWD/$so timeout 300 python scripts/kernel_crossover.py --kernels warp --tag $(basename $so .so) \
      --games ${GAMES:-pong_standin brix_standin target_shooter_level1 target_shooter_level3} --ns ${NS:-512 2048 4096} >> gpurun_out/ab_ff.jsonl 2>/dev/null
  done
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/ab_ff.jsonl"):
    r = json.loads(l); d[(r["game"], r["n"], r["tag"])].append((r["step_steps_per_s"], r["fused_steps_per_s"]))
for k in sorted(d):
    v = d[k]; print(f"{k[0]:22s} {k[1]:6d} {k[2]:12s} step {max(a for a, b in v):.4g} fused {max(b for a, b in v):.4g}")
PY
