#!/bin/bash
# ncu --set full of one step launch for every ab/*.so (GAME, ENVS), reports in gpurun_out/
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
GAME=${GAME:-pong_standin}; ENVS=${ENVS:-262144}
for so in ab/*.so; do
  nm=$(basename $so .so)
  PCMD="python bench.py --steps 3 --warmup 3 --envs $ENVS --game $GAME --no-sweep --no-e2e --no-cpu --no-fused"
  OCTAX_LIB=$PWD/$so timeout 300 $PCMD > gpurun_out/plain_$nm.log 2>&1 && \
  OCTAX_LIB=$PWD/$so timeout 600 ncu --set full --clock-control none --import-source on -k regex:octax_kernel -s 5 -c 1 \
     -o gpurun_out/abp_${GAME}_$nm -f $PCMD > gpurun_out/ncu_$nm.log 2>&1
  echo "$nm rc=$?"
done
