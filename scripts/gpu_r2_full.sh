#!/bin/bash
# round-2 evidence pass: GPU suite, smoke, ncu --set full of one headline step launch at 1M and
# 262,144 envs (summaries stamped with the device-code digest; latest_step_full.json feeds the
# bench's ALU / issue roofs), default bench line, ncu launch list of the same bench command,
# optional paper protocol (PROTOCOL=1)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
SO=paper_2510_01764_b200/liboctax.so
if [ -z "$SKIP_TESTS" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  tail -3 gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -1 gpurun_out/smoke.log
fi
for ENVS in 1048576 262144; do
  TAG=full_$ENVS
  PCMD="python bench.py --steps 3 --warmup 3 --envs $ENVS --no-sweep --no-e2e --no-cpu --no-fused"
  timeout 300 $PCMD > gpurun_out/plain_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:octax_kernel -s 5 -c 1 -o gpurun_out/$TAG -f $PCMD > gpurun_out/ncu_$TAG.log 2>&1
  echo "ncu $TAG rc=$?"
  python scripts/ncu_summary.py full gpurun_out/$TAG.ncu-rep gpurun_out/step_$TAG.json --envs $ENVS --game pong_standin --so $SO > /dev/null 2>&1
done
cp gpurun_out/step_full_1048576.json profiles/latest_step_full.json && echo "latest_step_full refreshed"
# the other games at configs[3]'s 262,144 envs (per-game instruction counts for the protocol rows)
for G in ${NCU_GAMES:-brix_standin target_shooter_level1 target_shooter_level2 target_shooter_level3}; do
  TAG=full_${G}_262144
  PCMD="python bench.py --steps 3 --warmup 3 --envs 262144 --game $G --no-sweep --no-e2e --no-cpu --no-fused"
  timeout 300 $PCMD > gpurun_out/plain_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:octax_kernel -s 5 -c 1 -o gpurun_out/$TAG -f $PCMD > gpurun_out/ncu_$TAG.log 2>&1
  echo "ncu $TAG rc=$?"
  python scripts/ncu_summary.py full gpurun_out/$TAG.ncu-rep gpurun_out/step_$TAG.json --envs 262144 --game $G --so $SO > /dev/null 2>&1
done
# the warp-per-env kernel (OCTAX_KERNEL_AUTO at n <= 4,096): configs[1]'s 4,096-env step
for G in ${WARP_GAMES:-pong_standin target_shooter_level3}; do
  TAG=warp_full_${G}_4096
  PCMD="python bench.py --steps 3 --warmup 3 --envs 4096 --game $G --no-sweep --no-e2e --no-cpu --no-fused"
  timeout 300 $PCMD > gpurun_out/plain_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:octax_warp_kernel -s 5 -c 1 -o gpurun_out/$TAG -f $PCMD > gpurun_out/ncu_$TAG.log 2>&1
  echo "ncu $TAG rc=$?"
  python scripts/ncu_summary.py full gpurun_out/$TAG.ncu-rep gpurun_out/$TAG.json --envs 4096 --game $G --so $SO > /dev/null 2>&1
done
if [ -n "$FUSED_NCU" ]; then  # one 100-step fused rollout launch (octax_kernel<2,1>) at 1M envs
  PCMD="python bench.py --steps 3 --warmup 3 --envs 1048576 --no-sweep --no-e2e --no-cpu"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:octax_kernel -s 8 -c 1 \
    -o gpurun_out/fused_1048576 -f $PCMD > gpurun_out/ncu_fused.log 2>&1; echo "ncu fused rc=$?"
  python scripts/ncu_summary.py full gpurun_out/fused_1048576.ncu-rep gpurun_out/fused_full_1048576.json \
    --envs 104857600 --game pong_standin --envs_per_launch 1048576 --so $SO > /dev/null 2>&1 && \
    cp gpurun_out/fused_full_1048576.json profiles/latest_fused_full.json
fi
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
if [ -n "$LAUNCHES" ]; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --no-sweep --no-fused > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
fi
if [ -n "$PROTOCOL" ]; then
  timeout 2400 python scripts/paper_protocol.py --out gpurun_out/paper_protocol > gpurun_out/protocol.log 2>&1; echo "protocol rc=$?"
fi
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
r = d["roofline"]
print("value %.4g ms/step %.4f bound %s frac %.3f fused %.4g e2e %.4g (link %.3f) full %.4g cpu %.3g" % (
    d["value"], d["ms_per_step"], r["bound"], r["frac"], d["fused"]["steps_per_s"], d["e2e"]["value"],
    d["e2e"]["link"]["frac"], d["e2e"]["full_obs"]["value"], d["cpu_baseline"]["value"]))
PY
