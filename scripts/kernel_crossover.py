#!/usr/bin/env python
"""Lane-per-env vs warp-per-env step kernel across batch sizes (octax_set_kernel): median
device time per octax_step (CUDA events, inputs resident) and per fused 100-step rollout step,
pong stand-in and the other bench games.  Prints one JSON line per (game, n, kernel, mode).

    python scripts/kernel_crossover.py [--games ...] [--ns 1024 4096 ...]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import workloads
    from paper_2510_01764_b200 import OctaxEnv
    ap = argparse.ArgumentParser()
    ap.add_argument("--games", nargs="*", default=["pong_standin", "brix_standin", "target_shooter_level1"])
    ap.add_argument("--ns", nargs="*", type=int, default=[512, 1024, 2048, 4096, 8192, 16384, 32768, 65536, 131072])
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--kernels", nargs="*", default=["lane", "warp"])
    ap.add_argument("--tag", default="")
    args = ap.parse_args()
    for game in args.games:
        rom, spec = workloads.game(game)
        for n in args.ns:
            for kernel in args.kernels:
                env = OctaxEnv(rom, spec, n, workloads.ENV_SEED, kernel=kernel)
                acts = torch.zeros(n, dtype=torch.int32, device="cuda")
                s = env.stream
                with torch.cuda.stream(s):
                    for t in range(10):
                        env.gen_actions(workloads.ACTION_SEED, t, acts)
                        env.step_into(acts, env.obs, env.reward, env.done)
                    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                    torch.cuda.synchronize()
                    ev[0].record(s)
                    for t in range(args.steps):
                        env.step_into(acts, env.obs, env.reward, env.done)
                    ev[1].record(s)
                    torch.cuda.synchronize()
                    ms = ev[0].elapsed_time(ev[1]) / args.steps
                    T = 100
                    r = torch.zeros(T * n, dtype=torch.float32, device="cuda")
                    d = torch.zeros(T * n, dtype=torch.uint8, device="cuda")
                    o = torch.zeros(n * 1024, dtype=torch.uint8, device="cuda")
                    env.rollout_into(T, o, r, d, aseed=workloads.ACTION_SEED, t0=0)
                    torch.cuda.synchronize()
                    ev[0].record(s)
                    env.rollout_into(T, o, r, d, aseed=workloads.ACTION_SEED, t0=T)
                    ev[1].record(s)
                    torch.cuda.synchronize()
                    fms = ev[0].elapsed_time(ev[1]) / T
                print(json.dumps({"tag": args.tag, "game": game, "n": n, "kernel": env.kernel, "step_ms": round(ms, 5),
                                  "step_steps_per_s": n / ms * 1e3, "fused_ms_per_step": round(fms, 5),
                                  "fused_steps_per_s": n / fms * 1e3}), flush=True)
                env.close()


if __name__ == "__main__":
    main()
