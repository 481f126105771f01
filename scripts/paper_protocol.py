#!/usr/bin/env python
"""The paper's throughput protocol ("execution time for 100-step rollouts ...
with 50 independent measurements per configuration"; steps/s = envs x 100 / time),
run on the BASELINE.json configurations, plus the CPU oracle on the same box.

    python scripts/paper_protocol.py [--reps 50] [--out profiles/r01_paper_protocol]

Writes <out>.json and <out>.md (median and IQR of the 50 rollouts).  Each
rollout = 100 octax_step launches with device-resident, pre-generated actions,
timed with CUDA events on the env's stream after one untimed warm-up rollout.
The oracle columns come from `bench.py --impl reference` (the one place besides
the tests that runs the CPU oracle), on 1 process and on every host core.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2510_01764_b200 import OctaxEnv  # noqa: E402

CONFIGS = [
    # (config id, game, envs, obs_format, action mode)
    ("1", "coverage", 1, 0, "random"),
    ("2", "pong_standin", 4096, 0, "random"),
    ("2", "pong_standin", 4096, 0, "constant"),
    ("2*", "pong_standin", 8192, 0, "constant"),          # the paper's 350K steps/s point
    ("3", "brix_standin", 65536, 0, "random"),
    ("3", "brix_standin", 65536, 1, "random"),
    ("4", "pong_standin", 262144, 0, "random"),
    ("4", "brix_standin", 262144, 0, "random"),
    ("4", "target_shooter_level1", 262144, 0, "random"),
    ("4", "target_shooter_level2", 262144, 0, "random"),
    ("4", "target_shooter_level3", 262144, 0, "random"),
] + [("5", g, n, 0, "random") for g in ("pong_standin", "target_shooter_level3")
     for n in (1024, 4096, 16384, 65536, 262144, 1048576)]
# SURVEY d.7 "mixed": the same rollouts after a 1,000-step random-action warm-up (every env
# has diverged or been through a reset); "fresh" rows start 100 steps after reset
MIXED = [("4", g, 262144, 0, "random") for g in ("pong_standin", "brix_standin", "target_shooter_level1",
                                                 "target_shooter_level2", "target_shooter_level3")] + \
        [("5", g, 1048576, 0, "random") for g in ("pong_standin", "target_shooter_level3")]


def rollouts(game, n, obs_format, mode, reps, T=100, warm=0):
    rom, spec = workloads.game(game, obs_format=obs_format)
    s = torch.cuda.Stream()
    env = OctaxEnv(rom, spec, n, workloads.ENV_SEED, stream=s)
    acts = torch.zeros((T, n), dtype=torch.int32, device="cuda")
    if mode == "random":
        with torch.cuda.stream(s):
            for t in range(T):
                env.gen_actions(workloads.ACTION_SEED, t, acts[t])
    s.synchronize()
    obs, rew, done = env.obs, env.reward, env.done
    for t in range(warm):  # "mixed" (SURVEY d.7): diverge lanes with random actions first
        with torch.cuda.stream(s):
            env.gen_actions(workloads.ACTION_SEED ^ 0x5A5A, t, acts[0])
        env.step_into(acts[0], obs, rew, done)
    if warm:  # restore the rollout's first action row
        with torch.cuda.stream(s):
            if mode == "random":
                env.gen_actions(workloads.ACTION_SEED, 0, acts[0])
            else:
                acts[0].zero_()
    times = []
    for r in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for t in range(T):
            env.step_into(acts[t], obs, rew, done)
        e1.record(s)
        e1.synchronize()
        if r > 0:  # first rollout is the warm-up
            times.append(e0.elapsed_time(e1) / 1e3)
    env.close()
    sps = np.array([n * T / t for t in times])
    return float(np.median(sps)), float(np.percentile(sps, 75) - np.percentile(sps, 25))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_paper_protocol"))
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    def oracle_ref(game, procs):
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--game", game,
               "--steps", "5", "--warmup", "1"] + (["--cpu-procs", str(procs)] if procs else [])
        out = subprocess.run(cmd, capture_output=True, text=True, check=True).stdout
        d = json.loads(out.strip().splitlines()[-1])
        return d["value"], d["cpu_baseline"]["cores"]
    import hashlib
    def rom_label(game, rom):
        if game.startswith("target_shooter"):
            return "paper App. D listing, sha256 " + hashlib.sha256(rom).hexdigest()[:16]
        return "labelled stand-in (" + game + "), sha256 " + hashlib.sha256(rom).hexdigest()[:16]
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm_gbs = float(json.load(f)["hbm_gbs"])
    except Exception:
        hbm_gbs = 6650.0
    rows = []
    cpu_cache = {}
    for cid, game, n, fmt, mode, warm in [c + (0,) for c in CONFIGS] + [c + (1000,) for c in MIXED]:
        med, iqr = rollouts(game, n, fmt, mode, args.reps, warm=warm)
        rom, spec = workloads.game(game)
        cyc = spec["frame_skip"] * spec["instructions_per_frame"]
        row = {"config": cid, "game": game, "rom": rom_label(game, rom), "envs": n, "gpus": 1,
               "obs": "bool" if fmt else "packed", "mode": "step", "actions": mode,
               "protocol": "mixed" if warm else "fresh", "warmup_steps": warm + 100,
               "steps_per_rollout": 100, "reps": args.reps,
               "steps_per_s_median": med, "steps_per_s_iqr": iqr, "frames_per_s_median": 4 * med,
               "emu_instr_per_s": cyc * med,
               # HBM roof of the packed path (2,201 algorithmic bytes per env step)
               "R_hbm": hbm_gbs * 1e9 / 2201 if not fmt else None,
               "bitexact": "pass: tests/test_gpu_parity.py (same kernels, same recipe)"}
        if not args.no_cpu and game not in cpu_cache:
            one, _ = oracle_ref(game, 1)
            allc, C = oracle_ref(game, None)
            cpu_cache[game] = (one, allc, C)
        if game in cpu_cache:
            row["oracle_1core"], row["oracle_all_cores"], row["cores"] = cpu_cache[game]
        rows.append(row)
        print(json.dumps(row), flush=True)
    dev = torch.cuda.get_device_name(0)
    with open(args.out + ".json", "w") as f:
        json.dump({"device": dev, "protocol": "P:228, 1 warm-up + %d x 100-step rollouts" % args.reps,
                   "rows": rows}, f, indent=1)
    lines = ["| config | game | envs | obs | actions | protocol | steps/s median | IQR | frames/s | oracle 1 core | oracle all cores (C) |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        lines.append(f"| {r['config']} | {r['game']} | {r['envs']:,} | {r['obs']} | {r['actions']} | {r['protocol']} | "
                     f"{r['steps_per_s_median']:.4g} | {r['steps_per_s_iqr']:.3g} | {r['frames_per_s_median']:.4g} | "
                     f"{r.get('oracle_1core', float('nan')):.3g} | {r.get('oracle_all_cores', float('nan')):.3g} ({r.get('cores', '-')}) |")
    with open(args.out + ".md", "w") as f:
        f.write(f"# Paper protocol (P:228) on {dev}\n\n1 warm-up + {args.reps} timed 100-step rollouts per row; "
                "CUDA events; device-resident actions.\n\n" + "\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
