#!/bin/bash
# the multi-rank bench path (2 ranks sharing one B200 over gloo) and the bounds-checked build
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --no-sweep --no-e2e > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err; echo "2-rank bench rc=$?"
cut -c1-300 gpurun_out/bench_2rank.json
bash scripts/gpu_checked.sh
