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


def regroup(game, warm=300, steps=24, cta=128):
    """SURVEY NEXT-2 (i) / VERDICT r1 #6: would regrouping a CTA's envs into warps by PC or by
    opcode class (an intra-CTA lane -> env permutation over the shared-memory-resident state)
    make warps uniform?  One CTA of `cta` envs (0..cta-1) is replayed cycle by cycle in the
    oracle; every warp-cycle is scored under three groupings of the CTA into warps of 32:
      identity      -- lane = env (the kernel as built);
      frame-sorted  -- at every frame boundary the envs are sorted by PC (then by opcode
                       class) and cut into warps; the grouping is held for the frame's cycles
                       (the regrouping a kernel could afford: one permutation per frame);
      cycle-sorted  -- re-sorted by the current PC at EVERY cycle (an upper bound no kernel
                       reaches: it would move every env's state every cycle).
    Scores: mean distinct PCs and distinct classes (high nibble; halted lanes = class -1) per
    warp-cycle, and the share of warp-cycles that are PC-uniform / class-uniform."""
    rom, spec = workloads.game(game)
    ipf, fs = spec["instructions_per_frame"], spec["frame_skip"]
    o = oracle.OracleEnv(rom, spec, cta, workloads.ENV_SEED)
    na = workloads.n_actions(spec)
    for t in range(warm):
        o.step(workloads.gen.actions(workloads.ACTION_SEED, t, cta, na))
    score = {g: {"pcs": 0.0, "cls": 0.0, "pc_uni": 0, "cls_uni": 0} for g in ("identity", "frame", "cycle")}
    wc = 0

    def peek():
        pcs, cls = np.zeros(cta, np.int64), np.zeros(cta, np.int64)
        for j in range(cta):
            f = oracle.canon_fields(o.get_state(j))
            pc, mem = int(f["PC"]), f["mem"]
            pcs[j] = pc
            cls[j] = -1 if f["halted"] or pc >= 0xFFF else int(mem[pc]) >> 4
        return pcs, cls

    def tally(name, order, pcs, cls):
        for w in range(cta // 32):
            idx = order[32 * w: 32 * w + 32]
            dp, dc = len(set(pcs[idx].tolist())), len(set(cls[idx].tolist()))
            sc = score[name]
            sc["pcs"] += dp
            sc["cls"] += dc
            sc["pc_uni"] += dp == 1
            sc["cls_uni"] += dc == 1

    ident = np.arange(cta)
    for t in range(warm, warm + steps):
        a = workloads.gen.actions(workloads.ACTION_SEED, t, cta, na)
        keys = [0 if x == 0 else 1 << spec["action_keys"][x - 1] for x in a]
        for _ in range(fs):
            pcs, cls = peek()
            frame_order = np.lexsort((cls, pcs))
            for k in range(ipf):
                if k:
                    pcs, cls = peek()
                tally("identity", ident, pcs, cls)
                tally("frame", frame_order, pcs, cls)
                tally("cycle", np.lexsort((cls, pcs)), pcs, cls)
                wc += cta // 32
                for j in range(cta):
                    o.run_cycles(j, 1, keys[j])
            for j in range(cta):
                o.tick_timers(j)
    return {g: {"distinct_pcs": v["pcs"] / wc, "distinct_classes": v["cls"] / wc,
                "pc_uniform": v["pc_uni"] / wc, "class_uniform": v["cls_uni"] / wc} for g, v in score.items()}


def sleepers(game, warm=300, steps=24, cta=128):
    """SURVEY NEXT-2 (ii) with (i): the frames an env sleeps through entirely -- halted, a
    self-jump, or a delay-poll loop (FX07; 3X00; 1NNN) entered with DT > 0 at the frame start (DT
    only changes at the frame's end, so the env provably loops until then) -- and how many whole
    warps a per-frame regrouping of a 128-env CTA by that status could skip: floor(sleepers / 32)
    per CTA-frame, against identity grouping (a warp skips only if all its 32 envs sleep)."""
    rom, spec = workloads.game(game)
    ipf, fs = spec["instructions_per_frame"], spec["frame_skip"]
    o = oracle.OracleEnv(rom, spec, cta, workloads.ENV_SEED)
    na = workloads.n_actions(spec)
    mem0 = [int(v) for v in oracle.canon_fields(o.get_state(0))["mem"]] + [0] * 8
    loops = _poll_loops(mem0)
    for t in range(warm):
        o.step(workloads.gen.actions(workloads.ACTION_SEED, t, cta, na))
    lane_frames = sleeping = warp_frames = skip_regroup = skip_ident = 0
    for t in range(warm, warm + steps):
        a = workloads.gen.actions(workloads.ACTION_SEED, t, cta, na)
        keys = [0 if x == 0 else 1 << spec["action_keys"][x - 1] for x in a]
        for _ in range(fs):
            sl = []
            for j in range(cta):
                f = oracle.canon_fields(o.get_state(j))
                pc, mem = int(f["PC"]), f["mem"]
                selfjump = pc < 0xFFF and (int(mem[pc]) << 8 | int(mem[pc + 1])) == (0x1000 | pc)
                sl.append(bool(f["halted"]) or selfjump or (pc in loops and int(f["DT"]) > 0))
            lane_frames += cta
            sleeping += sum(sl)
            warp_frames += cta // 32
            skip_regroup += sum(sl) // 32
            skip_ident += sum(all(sl[w * 32:(w + 1) * 32]) for w in range(cta // 32))
            for j in range(cta):
                o.run_cycles(j, ipf, keys[j])
                o.tick_timers(j)
    return {"sleeping_lane_frames": sleeping / lane_frames, "skippable_warp_frames_regrouped": skip_regroup / warp_frames,
            "skippable_warp_frames_identity": skip_ident / warp_frames}


def draw_traces(game, warm=300, steps=24, cta=128):
    """Per frame, per env, per instruction slot k < ipf: the rows the instruction at slot k draws
    (0 = not a DXYN).  An env's instruction stream does not depend on how its warp schedules
    it, so every scheduling policy below replays these same traces."""
    rom, spec = workloads.game(game)
    ipf, fs = spec["instructions_per_frame"], spec["frame_skip"]
    o = oracle.OracleEnv(rom, spec, cta, workloads.ENV_SEED)
    na = workloads.n_actions(spec)
    for t in range(warm):
        o.step(workloads.gen.actions(workloads.ACTION_SEED, t, cta, na))
    frames = []
    for t in range(warm, warm + steps):
        a = workloads.gen.actions(workloads.ACTION_SEED, t, cta, na)
        keys = [0 if x == 0 else 1 << spec["action_keys"][x - 1] for x in a]
        for _ in range(fs):
            fr = np.zeros((cta, ipf), np.int32)
            for j in range(cta):
                for k in range(ipf):
                    f = oracle.canon_fields(o.get_state(j))
                    pc, mem = int(f["PC"]), f["mem"]
                    word = (int(mem[pc]) << 8 | int(mem[pc + 1])) if pc < 0xFFF else 0
                    if word >> 12 == 0xD and not f["halted"]:  # clipped rows (A18), >= 1 marks a draw
                        fr[j, k] = max(1, min(word & 15, 32 - (int(f["V"][(word >> 4) & 15]) & 31)))
                    o.run_cycles(j, 1, keys[j])
                o.tick_timers(j)
            frames.append(fr)
    return frames


# warp instructions per warp-cycle, from profiles/r02_v42_source_attr_1M.md (pong, 1M envs):
# the interpreter core without the draw paths ~118 (rounded to 120; 80 as a what-if for a much
# cheaper core), and per DXYN dispatch, by the kernel's path choice: grouped ~65, single-row ~24,
# lane-parallel ~15 + 14 per row step, cooperative ~200, each + ~10 for the votes / reduce
def _draw_cost(rows):
    k, mx = len(rows), max(rows)
    if mx >= 3 and k * mx <= 32:
        return 10 + 65
    if mx == 1:
        return 10 + 25
    return 10 + (15 + 14 * mx if mx <= 8 else 200)


def _batched_frame(fr, core, K=None, W=None):
    """One warp's frame (fr: [32, ipf]) under draw batching: a lane reaching a DXYN waits (no
    effect, PC held) until the warp fires a batch -- when K lanes wait, a lane has waited W
    iterations, or no other unfinished lane can advance; K=None is the kernel as built (every
    DXYN drawn in the cycle it is reached).  The warp iterates until every lane has executed
    its ipf instructions.  Returns (iterations, draw dispatches, cost in warp instructions)."""
    n, ipf = fr.shape
    cnt, wait = np.zeros(n, np.int64), np.zeros(n, np.int64)
    it = dr = 0
    cost = 0.0
    while (cnt < ipf).any():
        it += 1
        cost += core
        live = np.nonzero(cnt < ipf)[0]
        rows = fr[live, cnt[live]]
        cnt[live[rows == 0]] += 1
        pend = live[rows != 0]
        if pend.size == 0:
            continue
        others = live.size - pend.size
        if K is None or pend.size >= K or others == 0 or wait[pend].max() + 1 >= W:
            cost += _draw_cost(fr[pend, cnt[pend]].tolist())
            dr += 1
            cnt[pend] += 1
            wait[pend] = 0
        else:
            wait[pend] += 1
    return it, dr, cost


BATCH_POLICIES = [(None, None), (4, 3), (8, 4), (8, 8), (16, 6), (32, 10 ** 9)]


def draw_batching(game, core=120.0, frames=None):
    """NEXT-2 / P:289 "adaptive batching", read as batching the DXYN draws of a warp: lanes that
    reach a draw wait so that one draw dispatch serves several of them.  Cost of each policy
    relative to the kernel as built, over the 4 warps of one 128-env CTA."""
    frames = draw_traces(game) if frames is None else frames
    out = {}
    for pol in BATCH_POLICIES:
        tot = np.zeros(3)
        for fr in frames:
            for w in range(fr.shape[0] // 32):
                tot += _batched_frame(fr[32 * w: 32 * w + 32], core, *pol)
        out[pol] = tot
    base = out[(None, None)][2]
    return {pol: {"iterations": int(v[0]), "draws": int(v[1]), "rel_cost": v[2] / base} for pol, v in out.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_workload_structure.md"))
    ap.add_argument("--games", nargs="*", default=GAMES)
    ap.add_argument("--regroup-out", default=None,
                    help="also write the NEXT-2 regrouping study (regroup()) to this file")
    ap.add_argument("--batching-out", default=None,
                    help="write the NEXT-2 draw-batching study (draw_batching()) to this file")
    args = ap.parse_args()
    if args.batching_out:
        bl = ["| game | policy (fire at K waiting / W iterations) | warp iterations | draw dispatches | "
              "cost, core 120 | cost, core 80 |", "|---|---|---|---|---|---|"]
        for g in args.games:
            tr = draw_traces(g)
            r120, r80 = draw_batching(g, 120.0, tr), draw_batching(g, 80.0, tr)
            for pol in BATCH_POLICIES:
                name = "as built (draw when reached)" if pol[0] is None else \
                    ("K=32 (all wait)" if pol[1] > 10 ** 6 else f"K={pol[0]}, W={pol[1]}")
                v = r120[pol]
                bl.append(f"| {g} | {name} | {v['iterations']} | {v['draws']} | {v['rel_cost']:.3f} | "
                          f"{r80[pol]['rel_cost']:.3f} |")
                print(bl[-1], flush=True)
        with open(args.batching_out, "w") as f:
            f.write("# NEXT-2 draw-batching study (oracle traces of one 128-env CTA, random actions)\n\n"
                    "Generated by `python -m tests.tools.workload_structure --batching-out ...` "
                    "(`draw_batching()`): 24 steps after a 300-step warm-up.  A lane that reaches a "
                    "DXYN waits until its warp fires a batched draw; the warp iterates until every lane "
                    "has run its ipf instructions.  Cost = warp iterations x core + draw dispatches x "
                    "path cost (warp instructions, model constants in the tool, from "
                    "`profiles/r02_v42_source_attr_1M.md`), relative to the kernel as built; the gating "
                    "of waiting lanes is not even charged.\n\n" + "\n".join(bl) + "\n")
        return
    if args.regroup_out:
        rl = ["| game | grouping | distinct PCs / warp-cycle | distinct classes / warp-cycle | "
              "PC-uniform warp-cycles | class-uniform warp-cycles |", "|---|---|---|---|---|---|"]
        for g in args.games:
            r = regroup(g)
            for name, v in r.items():
                rl.append(f"| {g} | {name} | {v['distinct_pcs']:.2f} | {v['distinct_classes']:.2f} | "
                          f"{100 * v['pc_uniform']:.1f}% | {100 * v['class_uniform']:.1f}% |")
                print(rl[-1], flush=True)
        rl += ["", "| game | env-frames slept through entirely | warp-frames skippable, identity grouping | "
               "warp-frames skippable, regrouped by sleep status per frame |", "|---|---|---|---|"]
        for g in args.games:
            z = sleepers(g)
            rl.append(f"| {g} | {100 * z['sleeping_lane_frames']:.1f}% | {100 * z['skippable_warp_frames_identity']:.1f}% | "
                      f"{100 * z['skippable_warp_frames_regrouped']:.1f}% |")
            print(rl[-1], flush=True)
        with open(args.regroup_out, "w") as f:
            f.write("# NEXT-2 regrouping study (oracle replay of one 128-env CTA, random actions)\n\n"
                    "Generated by `python -m tests.tools.workload_structure --regroup-out ...` "
                    "(`regroup()`): 24 steps after a 300-step warm-up; identity = lane is env (the "
                    "kernel as built), frame = envs sorted by (PC, class) once per frame and held "
                    "for its cycles, cycle = re-sorted every cycle (unreachable upper bound).\n\n"
                    + "\n".join(rl) + "\n")
        return
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
