#!/usr/bin/env python
"""Cost of the in-step auto-reset with startup segments (build-plan item 4h):
env steps/s of the brix stand-in (random actions: episodes end, ~17 per 1,000 steps per env)
at 1M envs without startup segments and with S startup frames after every reset.

    python scripts/reset_cost.py [--envs N] [--frames 0 4 16 64]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2510_01764_b200 import OctaxEnv  # noqa: E402


def rate(n, frames, steps=20, warm=30):
    startup = [(1 << 4, frames)] if frames else []
    rom, spec = workloads.game("brix_standin", startup=startup, max_episode_steps=200)
    s = torch.cuda.Stream()
    env = OctaxEnv(rom, spec, n, workloads.ENV_SEED, stream=s)
    acts = torch.empty((warm + steps, n), dtype=torch.int32, device="cuda")
    with torch.cuda.stream(s):
        for t in range(warm + steps):
            env.gen_actions(workloads.ACTION_SEED, t, acts[t])
    obs, rew, done = env.obs, env.reward, env.done
    for t in range(warm):
        env.step_into(acts[t], obs, rew, done)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    resets = torch.zeros((), dtype=torch.int64, device="cuda")
    with torch.cuda.stream(s):
        ev0.record(s)
        for t in range(warm, warm + steps):
            env.step_into(acts[t], obs, rew, done)
        ev1.record(s)
    s.synchronize()
    ms = ev0.elapsed_time(ev1)
    st, _ = env.stats()
    env.close()
    return n * steps / (ms / 1e3), int(st[1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=1 << 20)
    ap.add_argument("--frames", type=int, nargs="*", default=[0, 4, 16, 64])
    a = ap.parse_args()
    rows = []
    for f in a.frames:
        v, eps = rate(a.envs, f)
        rows.append({"startup_frames": f, "env_steps_per_s": v, "episodes_finished": eps})
        print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
