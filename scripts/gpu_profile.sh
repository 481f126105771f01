#!/bin/bash
# profile pass: fixed tests, plain bench, ncu launch list (default bench cmd), ncu --set full on one step launch
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "expression" -p no:cacheprovider > gpurun_out/pytest_expr.log 2>&1; tail -3 gpurun_out/pytest_expr.log
CMD="python bench.py --steps 20 --warmup 5"
timeout 600 $CMD > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
PCMD="python bench.py --steps 3 --warmup 3 --envs 262144 --no-sweep --no-e2e --no-cpu --no-fused"
timeout 300 $PCMD > gpurun_out/plain_prof.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:octax_kernel -s 5 -c 1 -o gpurun_out/prof_step -f $PCMD > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
cut -c1-300 gpurun_out/bench_plain.json
