#!/bin/bash
# A/B timing of kernel variants on one box: ab/*.so built locally with
#   python paper_2510_01764_b200/build.py --out ab/<name>.so
# Each variant is timed ROUNDS times, interleaved, per game.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
ROUNDS=${ROUNDS:-3}
GAMES=${GAMES:-"pong_standin brix_standin target_shooter_level1"}
for r in $(seq $ROUNDS); do
  for so in ab/*.so; do
    for g in $GAMES; do
      v=$(OCTAX_LIB=$PWD/$so timeout 300 python bench.py --no-e2e --no-cpu --no-sweep --no-fused --game $g --steps 20 --warmup 5 $EXTRA 2>/dev/null \
          | python -c "import json,sys; print('%.4g' % json.loads(sys.stdin.read())['value'])")
      echo "round $r $(basename $so) $g $v"
    done
  done
done | tee gpurun_out/ab.log
