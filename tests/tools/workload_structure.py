#!/usr/bin/env python
"""Workload structure of the bench games, measured with the CPU oracle (SURVEY §8(d)
d.1 "record the workload structure the oracle can measure cheaply" and d.7's
divergence model).  Test infrastructure: lives under tests/ because it runs oracle/.

    python -m tests.tools.workload_structure [--out profiles/r01_workload_structure.md]

Per game (random actions, Philox domain 1):
  * opcode-class histogram (share of executed instructions by high nibble),
    DXYN per step, sprite rows per DXYN, episodes finished per 1000 env steps
    -- from the oracle's per-VM counters over 256 envs x 400 steps;
  * cycle-level lockstep structure of one 32-lane warp (envs 0..31) over 40 steps
    after a 300-step warm-up: distinct PCs per warp-cycle, the share of lane-cycles
    spent in a delay-poll loop (FX07; 3X00; 1NNN back, with DT > 0) or a self-jump,
    and the share of cycles that end a frame with ALL 32 lanes idle -- the only
    cycles a warp-uniform idle-loop fast-forward could skip.
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads  # noqa: E402

GAMES = ["pong_standin", "brix_standin", "target_shooter_level1", "target_shooter_level2",
         "target_shooter_level3"]


def _poll_loops(mem):
    """Addresses of delay-poll loops A: FX07 ; 3X00 ; 1A (Octo's wait-delay)."""
    s = set()
    w = lambda a: mem[a] << 8 | mem[a + 1]  # noqa: E731
    for a in range(0x200, 0xFF9):
        w0, w1, w2 = w(a), w(a + 2), w(a + 4)
        if (w0 & 0xF0FF) == 0xF007 and (w1 & 0xF0FF) == 0x3000 and (w1 >> 8) & 15 == (w0 >> 8) & 15 \
                and w2 == (0x1000 | a):
            s.update((a, a + 2, a + 4))
    return s


def counters(game, n=128, steps=300):
    rom, spec = workloads.game(game)
    o = oracle.OracleEnv(rom, spec, n, workloads.ENV_SEED)
    na = workloads.n_actions(spec)
    eps = 0
    c = np.zeros(17, np.float64)
    for t in range(steps):                     # the oracle's counters cover the last step
        eps += int(o.step(workloads.gen.actions(workloads.ACTION_SEED, t, n, na))[2].sum())
        c += np.sum([o.counters(j) for j in range(n)], axis=0)
    cls, rows = c[:16], c[16]
    return {"hist": cls / cls.sum(), "draws_per_step": cls[0xD] / (n * steps),
            "rows_per_draw": rows / max(cls[0xD], 1), "episodes_per_1k": 1000.0 * eps / (n * steps)}


def lockstep(game, warm=300, steps=40):
    rom, spec = workloads.game(game)
    n, ipf, fs = 32, spec["instructions_per_frame"], spec["frame_skip"]
    o = oracle.OracleEnv(rom, spec, n, workloads.ENV_SEED)
    na = workloads.n_actions(spec)
    mem0 = [int(v) for v in oracle.canon_fields(o.get_state(0))["mem"]] + [0] * 8
    loops = _poll_loops(mem0)
    for t in range(warm):
        o.step(workloads.gen.actions(workloads.ACTION_SEED, t, n, na))
    pcs, idle_lc, lc, tail, cyc = [], 0, 0, 0, 0
    paths = {"grouped": 0, "single-row": 0, "lane-parallel": 0, "cooperative": 0}
    for t in range(warm, warm + steps):
        a = workloads.gen.actions(workloads.ACTION_SEED, t, n, na)
        keys = [0 if x == 0 else 1 << spec["action_keys"][x - 1] for x in a]
        for _ in range(fs):
            idle = np.zeros((ipf, n), bool)
            for k in range(ipf):
                pc_k, rows = [], []
                for j in range(n):
                    f = oracle.canon_fields(o.get_state(j))
                    pc = int(f["PC"])
                    mem = f["mem"]
                    word = (int(mem[pc]) << 8 | int(mem[pc + 1])) if pc < 0xFFF else 0
                    if word >> 12 == 0xD and not f["halted"]:   # DXYN rows this cycle (clipped, A18)
                        rows.append(min(word & 15, 32 - (int(f["V"][(word >> 4) & 15]) & 31)))
                    selfjump = pc < 0xFFF and (int(mem[pc]) << 8 | int(mem[pc + 1])) == (0x1000 | pc)
                    idle[k, j] = bool(f["halted"]) or selfjump or (pc in loops and int(f["DT"]) > 0)
                    pc_k.append(pc)
                    o.run_cycles(j, 1, keys[j])
                pcs.append(len(set(pc_k)))
                if rows:   # the kernel's per-warp DXYN choice (octax_kernels.cu, cycle())
                    mx, kd = max(rows), sum(1 for r in rows if r)
                    paths["grouped" if mx >= 3 and kd <= 32 // mx else "single-row" if mx == 1
                          else "lane-parallel" if mx <= 8 else "cooperative"] += 1
            for j in range(n):
                o.tick_timers(j)
            idle_lc += int(idle.sum())
            lc += idle.size
            all_idle = idle.all(axis=1)
            for k in range(ipf - 1, -1, -1):
                if not all_idle[k]:
                    break
                tail += 1
            cyc += ipf
        # step-end bookkeeping (reward / termination / reset) is skipped here: the
        # run_cycles hooks do not evaluate expressions; 40 steps rarely end an episode
    return {"distinct_pcs": float(np.mean(pcs)), "idle_lane_cycles": idle_lc / lc,
            "warp_skippable_cycles": tail / cyc, "draw_paths": {k: v / cyc for k, v in paths.items()}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_workload_structure.md"))
    ap.add_argument("--games", nargs="*", default=GAMES)
    args = ap.parse_args()
    lines = ["| game | top classes (share of instructions) | DXYN/step | rows/DXYN | episodes/1k steps | "
             "distinct PCs per warp-cycle | idle lane-cycles | all-32-idle frame-tail cycles | "
             "warp-cycles by DXYN path (grouped / single-row / lane-parallel / cooperative) |",
             "|---|---|---|---|---|---|---|---|---|"]
    for g in args.games:
        c, s = counters(g), lockstep(g)
        top = ", ".join(f"{k:X}: {100 * c['hist'][k]:.0f}%" for k in np.argsort(-c["hist"])[:6])
        lines.append(f"| {g} | {top} | {c['draws_per_step']:.2f} | {c['rows_per_draw']:.2f} | "
                     f"{c['episodes_per_1k']:.2f} | {s['distinct_pcs']:.1f} | {100 * s['idle_lane_cycles']:.1f}% | "
                     f"{100 * s['warp_skippable_cycles']:.2f}% | "
                     + " / ".join(f"{100 * v:.0f}%" for v in s["draw_paths"].values()) + " |")
        print(lines[-1], flush=True)
    hdr = ("# Workload structure (oracle, random actions)\n\n"
           "Generated by `python -m tests.tools.workload_structure`.  Class = high nibble of the "
           "opcode; lockstep columns are one warp (envs 0..31) over 40 steps after a 300-step warm-up.\n\n")
    with open(args.out, "w") as f:
        f.write(hdr + "\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
