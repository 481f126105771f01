#!/bin/bash
# ncu --set full on one step launch (after a plain run of the same command exits 0)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
ENVS=${ENVS:-1048576}
TAG=${TAG:-prof}
PCMD="python bench.py --steps 3 --warmup 3 --envs $ENVS --no-sweep --no-e2e --no-cpu --no-fused"
timeout 300 $PCMD > gpurun_out/plain_prof.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:octax_kernel -s 5 -c 1 -o gpurun_out/$TAG -f $PCMD > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full.log
