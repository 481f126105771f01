#!/bin/bash
# e2e (host-buffer) throughput of ab/*.so: bench.py's e2e key, interleaved rounds
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for r in $(seq ${ROUNDS:-3}); do
  for so in ab/*.so; do
    OCTAX_LIB=$PWD/$so timeout 300 python bench.py --no-cpu --no-sweep --no-fused --steps 10 --warmup 3 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('round $r $(basename $so) frame %.4g (%.3f) full %.4g (%.3f)' % (e['value'], e['link']['frac'], e['full_obs']['value'], e['full_obs']['link']['frac']))"
  done
done | tee gpurun_out/ab_e2e.log
