#!/bin/bash
# one ncu --set full capture of the warp-per-env step kernel (pong stand-in, 4,096 envs)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
python scripts/warp_profile_run.py pong_standin ${N:-4096} warp ${MODE:-step} || exit 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:octax_warp_kernel -s ${SKIP:-3} -c 1 \
  -o gpurun_out/warp_${MODE:-step}_${N:-4096} -f python scripts/warp_profile_run.py pong_standin ${N:-4096} warp ${MODE:-step} > gpurun_out/warp_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/warp_ncu.log
python scripts/ncu_summary.py full gpurun_out/warp_${MODE:-step}_${N:-4096}.ncu-rep gpurun_out/warp_${MODE:-step}_${N:-4096}.json \
  --envs $(( ${N:-4096} * $( [ "${MODE:-step}" = fused ] && echo 100 || echo 1 ) )) --game pong_standin --so paper_2510_01764_b200/liboctax.so > /dev/null 2>&1
