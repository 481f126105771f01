"""bench.py's multi-rank path on the GPU (-m gpu): torchrun with 2 ranks.  On a one-GPU box the
ranks share the device and bench.py selects the gloo backend (--dist-backend auto); the host
logic -- contiguous global-id shards, the per-rollout int64[4] all-reduce inside
the timed region, max-over-ranks timing, the state-digest reduction -- is the same as under
NCCL.  Trajectories are keyed by global env id (A13), so:
  * the 2-rank job over 2 x n envs reproduces a 1-rank job over 2n envs exactly: same reduced
    episode statistics, same all-rank digest sum;
  * rank 0's shard digest (global ids [0, n)) equals a 1-rank job over n envs."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N = 4096
COMMON = ["--game", "brix_standin", "--steps", "20", "--warmup", "3", "--rollout", "8", "--max-episode-steps", "7",
          "--no-sweep", "--no-e2e", "--no-cpu", "--no-fused"]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _line(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_two_rank_bench_matches_single_rank():
    one_2n = _line([sys.executable, "bench.py", "--envs", str(2 * N), *COMMON])
    one_n = _line([sys.executable, "bench.py", "--envs", str(N), *COMMON])
    two = _line([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                 "--master-addr", "127.0.0.1", "--master-port", str(_port()),
                 "bench.py", "--gpus", "2", "--envs", str(N), *COMMON])
    assert two["n_gpus"] == 2 and two["config"]["global_envs"] == 2 * N
    assert two["dist"]["world"] == 2 and two["dist"]["backend"] in ("gloo", "nccl")
    # 20 timed steps, rollout 8: all-reduces after steps 8, 16 and the last one
    assert two["dist"]["stats_allreduces_in_timed_region"] == 3
    assert two["stats"] == one_2n["stats"] and two["stats"][1] > 0      # episodes ended and reset
    assert two["stats"][2] == 2 * N * 23                                # (warmup + steps) x envs
    assert two["state_digest"]["all_ranks_sum"] == one_2n["state_digest"]["all_ranks_sum"]
    assert two["state_digest"]["rank0_shard_sum"] == one_n["state_digest"]["rank0_shard_sum"]
    assert two["value"] > 0 and two["ms_per_step"] > 0
