#!/usr/bin/env python
"""A few steps of one game on the forced warp-per-env kernel (ncu target; not a bench)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
from paper_2510_01764_b200 import OctaxEnv

game = sys.argv[1] if len(sys.argv) > 1 else "pong_standin"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
kernel = sys.argv[3] if len(sys.argv) > 3 else "warp"
rom, spec = workloads.game(game)
env = OctaxEnv(rom, spec, n, workloads.ENV_SEED, kernel=kernel)
acts = torch.zeros(n, dtype=torch.int32, device="cuda")
mode = sys.argv[4] if len(sys.argv) > 4 else "step"
if mode == "fused":  # 4 fused 100-step rollouts (no per-step obs kept)
    r = torch.zeros(100 * n, dtype=torch.float32, device="cuda")
    d = torch.zeros(100 * n, dtype=torch.uint8, device="cuda")
    for k in range(4):
        env.rollout_into(100, env.obs, r, d, aseed=workloads.ACTION_SEED, t0=100 * k)
else:
    for t in range(6):
        env.gen_actions(workloads.ACTION_SEED, t, acts)
        env.step_into(acts, env.obs, env.reward, env.done)
torch.cuda.synchronize()
print("ok", env.kernel)
