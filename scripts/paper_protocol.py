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


def rollouts(game, n, obs_format, mode, reps, T=100, warm=0, launch="step"):
    """Median / IQR steps/s of `reps` timed 100-step rollouts after one untimed one.  launch:
    "step" = 100 octax_step launches; "graph" = the same 100 launches captured in one CUDA graph;
    "fused" = one octax_rollout launch (in-kernel actions for random mode; a constant-action
    rollout passes the zero [T][n] action buffer)."""
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
    g = None
    if launch == "graph":
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for t in range(T):
                env.step_into(acts[t], obs, rew, done)
    times = []
    for r in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        if launch == "graph":
            with torch.cuda.stream(s):
                g.replay()
        elif launch == "fused":
            with torch.cuda.stream(s):
                env.rollout_into(T, obs, rew, done, actions=None if mode == "random" else acts,
                                 aseed=workloads.ACTION_SEED, t0=0)
        else:
            for t in range(T):
                env.step_into(acts[t], obs, rew, done)
        e1.record(s)
        e1.synchronize()
        if r > 0:  # first rollout is the warm-up
            times.append(e0.elapsed_time(e1) / 1e3)
    del g
    kernel = env.kernel  # OCTAX_KERNEL_AUTO's choice: warp-per-env for n <= 4,096
    env.close()
    sps = np.array([n * T / t for t in times])
    return float(np.median(sps)), float(np.percentile(sps, 75) - np.percentile(sps, 25)), kernel


# SURVEY d.8 "bitexact, n_envs_checked, steps_checked": the GPU parity test that covers each
# configuration with the same kernels and input recipe (its pass/fail is read from the pytest log
# of the same box run, gpurun_out/pytest_gpu.log, when present)
BITEXACT = {
    "1": ("tests/test_gpu_parity.py::test_coverage_rom_n1_1000_steps_full_state_every_step", 1, 1000),
    "2": ("tests/test_gpu_kernels.py::test_config2_pong_4096_sampled_parity (every env, warp kernel as AUTO runs it) + "
          "tests/test_gpu_rollout.py::test_rollout_equals_steps_on_gpu_at_4096", 4096, 200),
    "2*": ("tests/test_gpu_parity.py::test_game_parity[pong_standin-300]", 300, 300),
    "3": ("tests/test_gpu_parity.py::test_game_parity[brix_standin-257] + test_bool_obs_startup_and_truncation_parity", 257, 300),
    "4": ("tests/test_gpu_parity.py::test_config4_sampled_parity_1000_steps (64 sampled envs per game)", 64, 1000),
    "5": ("tests/test_gpu_parity.py::test_full_size_sampled_parity (64 sampled envs at 1M) + "
          "tests/test_gpu_rollout.py::test_rollout_1M_sampled_parity_and_step_equivalence", 64, 100),
}


def pytest_status(tests: str):
    """pass / FAIL for the row's own parity tests, from the GPU suite's log of the same box run."""
    try:
        log = open(os.path.join(ROOT, "gpurun_out", "pytest_gpu.log")).read()
    except OSError:
        return "not run on this box"
    if "passed" not in log:
        return "no result"
    failed = [l.split("::")[-1].split("[")[0] for l in log.splitlines() if l.startswith("FAILED ")]
    bad = [f for f in failed if f in tests]
    return "FAIL: " + ", ".join(bad) if bad else "pass"


def ncu_model(game, n, kernel="lane"):
    """I_step, ALU-pipe instructions, eta and DRAM bytes per env step from an ncu capture of THIS
    build (device-code digest) of the kernel that ran the row (lane-per-env: step_full*.json;
    warp-per-env: warp_full*.json) for this game: the one at this env count if there is one, else
    the game's capture at another count (instructions per env step do not depend on n: 363.2 at 1M
    vs 363.3 at 262K for kernel v35; DRAM bytes do, below ~1e5 envs the state stays in L2)."""
    import glob
    from paper_2510_01764_b200 import octax
    from paper_2510_01764_b200.build import device_code_digest
    have = device_code_digest(octax.SO_PATH)
    caps = []
    pat = "warp_full" if kernel == "warp" else "step_full"
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", f"*{pat}*.json")) +
                    glob.glob(os.path.join(ROOT, "gpurun_out", f"{pat}*.json"))):
        try:
            j = json.load(open(f))
        except Exception:
            continue
        if j.get("sass_sha256") == have and j.get("game") == game:
            caps.append((j.get("envs") != n, f, j))
    for _, f, j in sorted(caps, key=lambda c: c[0]):
        if True:
            return {"I_step_warp": j.get("warp_instr_per_env_step"),
                    "I_step_thread": (j.get("warp_instr_per_env_step") or 0) * 32 * (j.get("warp_exec_efficiency") or 0),
                    "alu_warp_instr_per_env_step": j.get("alu_warp_instr_per_env_step"),
                    "eta": j.get("warp_exec_efficiency"),
                    "dram_bytes_per_step": j.get("dram_bytes_per_env_step") if j.get("envs") == n else None,
                    "source": os.path.relpath(f, ROOT) + ("" if j.get("envs") == n else
                                                          f" (capture at {j.get('envs')} envs)")}
    return None


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
    cpu_model = ""
    try:
        with open("/proc/cpuinfo") as f:
            cpu_model = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except Exception:
        pass
    from bench import ClockSampler
    jobs = []
    for cid, game, n, fmt, mode, warm in [c + (0,) for c in CONFIGS] + [c + (1000,) for c in MIXED]:
        launches = ["step", "fused"]
        if n <= 65536 and not warm:
            launches.append("graph")
        jobs += [(cid, game, n, fmt, mode, warm, ln) for ln in launches]
    for cid, game, n, fmt, mode, warm, launch in jobs:
        with ClockSampler(0) as clk:
            med, iqr, kernel = rollouts(game, n, fmt, mode, args.reps, warm=warm, launch=launch)
        ck = clk.summary()
        f_sm = (ck["sm_mhz"] or 1965.0) * 1e6
        rom, spec = workloads.game(game)
        cyc = spec["frame_skip"] * spec["instructions_per_frame"]
        nm = ncu_model(game, n, kernel) if fmt == 0 else None  # fused: the step kernel's counts (an upper bound)
        # SURVEY d.2 roofs: issue = 148 SMs x 4 schedulers x 1 warp instr / cycle; ALU pipe = 148 x 4 x
        # 1 warp instr / 2 cycles; each / the measured warp instructions per env step
        R_issue = 148 * 4 * f_sm / nm["I_step_warp"] if nm and nm["I_step_warp"] else None
        R_alu = 148 * 4 * 0.5 * f_sm / nm["alu_warp_instr_per_env_step"] if nm and nm["alu_warp_instr_per_env_step"] else None
        # algorithmic B / env step: step mode 2,201; fused 1,797 (no state round trip,
        # no framebuffer TMA read, actions generated in the kernel)
        R_hbm = hbm_gbs * 1e9 / (1797 if launch == "fused" else 2201) if not fmt else None
        roofs = {k: v for k, v in (("issue", R_issue), ("alu", R_alu), ("hbm", R_hbm)) if v}
        binding = min(roofs, key=roofs.get) if roofs else None
        bt, be, bs = BITEXACT.get(cid, ("", 0, 0))
        if launch == "fused":
            bt += (" + tests/test_gpu_rollout.py (test_rollout_games_parity, test_rollout_generated_actions_parity, "
                   "test_rollout_equals_steps_on_gpu_at_4096, test_rollout_1M_sampled_parity_and_step_equivalence)")
        row = {"config": cid, "game": game, "rom": rom_label(game, rom), "envs": n, "gpus": 1, "kernel": kernel,
               "obs": "bool" if fmt else "packed", "mode": launch, "actions": mode,
               "protocol": "mixed" if warm else "fresh", "warmup_steps": warm + 100,
               "steps_per_rollout": 100, "reps": args.reps,
               "steps_per_s_median": med, "steps_per_s_iqr": iqr, "frames_per_s_median": 4 * med,
               "emu_instr_per_s": cyc * med,
               "sm_clock_mhz_during": ck["sm_mhz"], "clock_reasons": ck["reasons"],
               "dram_bytes_per_step_ncu": nm and nm["dram_bytes_per_step"], "I_step_ncu": nm and nm["I_step_thread"],
               "I_step_warp_ncu": nm and nm["I_step_warp"], "eta_ncu": nm and nm["eta"],
               "ncu_source": nm["source"] if nm else "no ncu capture of this build at this game / env count",
               "R_issue": R_issue, "R_alu": R_alu, "R_hbm": R_hbm, "binding": binding,
               "frac_binding": med / roofs[binding] if binding else None,
               "bitexact": pytest_status(bt), "bitexact_test": bt, "n_envs_checked": be, "steps_checked": bs,
               "cpu_model": cpu_model,
               **({"obs_note": "fused + bool: packed obs every step, bool expansion of the last step only "
                               "(stride-0 rollout: intermediate obs are overwritten)"} if launch == "fused" and fmt else {})}
        # self-consistency: steps/s recomputes from the row's own fields
        assert abs(row["frames_per_s_median"] - 4 * row["steps_per_s_median"]) < 1e-6 * row["frames_per_s_median"]
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
    lines = ["| config | game | envs | kernel | obs | mode | actions | protocol | steps/s median | IQR | frames/s | SM MHz | "
             "binding roof (frac) | bitexact (envs x steps) | oracle 1 core | oracle all cores (C) |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        roof = f"{r['binding']} ({r['frac_binding']:.2f})" if r["binding"] else "-"
        mode = r["mode"] + (" (bool expanded for the last step)" if r.get("obs_note") else "")
        lines.append(f"| {r['config']} | {r['game']} | {r['envs']:,} | {r['kernel']} | {r['obs']} | {mode} | {r['actions']} | "
                     f"{r['protocol']} | {r['steps_per_s_median']:.4g} | {r['steps_per_s_iqr']:.3g} | "
                     f"{r['frames_per_s_median']:.4g} | {r['sm_clock_mhz_during']} | {roof} | "
                     f"{r['bitexact']} ({r['n_envs_checked']} x {r['steps_checked']}) | "
                     f"{r.get('oracle_1core', float('nan')):.3g} | {r.get('oracle_all_cores', float('nan')):.3g} ({r.get('cores', '-')}) |")
    with open(args.out + ".md", "w") as f:
        f.write(f"# Paper protocol (P:228) on {dev}, host CPU {cpu_model}\n\n1 warm-up + {args.reps} timed 100-step "
                "rollouts per row; CUDA events; device-resident actions (fused: generated in the kernel).  Modes "
                "(SURVEY d.8): step = 100 octax_step launches, graph = the same launches in one CUDA graph, "
                "fused = one octax_rollout launch.  Kernel = OCTAX_KERNEL_AUTO's choice (warp-per-env for n <= "
                "4,096, lane-per-env above).  Roofs (SURVEY d.2): issue / ALU pipe from the ncu capture of "
                "this build's kernel at the row's game and env count, HBM from 2,201 algorithmic B per env step; "
                "the full d.8 row is in the .json.\n\n" + "\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
