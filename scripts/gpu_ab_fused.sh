#!/bin/bash
# A/B of ab/*.so in the fused rollout mode (bench.py's `fused` key: 100-step rollouts at 1M envs),
# parity-gated like gpu_ab_parity.sh; step-mode values printed alongside
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for so in ab/*.so; do
  OCTAX_LIB=$PWD/$so timeout 900 python -m pytest tests/test_gpu_rollout.py tests/test_gpu_parity.py -m gpu -q -x \
     -p no:cacheprovider -k "${PARITY_K:-rollout or game_parity or quirk_parity}" > gpurun_out/parity_$(basename $so .so).log 2>&1
  echo "$(basename $so) parity rc=$? $(tail -1 gpurun_out/parity_$(basename $so .so).log)"
done
for r in $(seq ${ROUNDS:-2}); do
  for g in ${GAMES:-pong_standin brix_standin target_shooter_level3}; do
    for so in ab/*.so; do
      OCTAX_LIB=$PWD/$so timeout 300 python bench.py --no-e2e --no-cpu --no-sweep --no-fused-noobs --game $g --steps 20 --warmup 5 2>/dev/null \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('round $r $(basename $so) $g step %.4g fused %.4g' % (d['value'], d['fused']['steps_per_s']))"
    done
  done
done | tee gpurun_out/ab_fused.log
