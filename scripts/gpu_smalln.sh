#!/bin/bash
# CTA-size variants (ab/*.so) at small env counts: step-mode launches, interleaved
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for r in 1 2; do
  for n in ${NS:-1024 4096 16384 65536}; do
    for so in ab/*.so; do
      v=$(OCTAX_LIB=$PWD/$so timeout 300 python bench.py --envs $n --steps 40 --warmup 5 --no-sweep --no-e2e --no-cpu --no-fused ${EXTRA} 2>/dev/null \
          | python -c "import json,sys; print('%.4g' % json.loads(sys.stdin.read())['value'])")
      echo "round $r n=$n $(basename $so) $v"
    done
  done
done | tee gpurun_out/smalln.log
