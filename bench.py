#!/usr/bin/env python
"""Benchmark of the batched Octax environment step (BASELINE.json metric:
env steps/s and frames/s vs #parallel envs, 1/2/4/8 B200).

Default workload (N=1): the per-GPU slice of BASELINE configs[4] -- 1,048,576
envs per GPU (the north-star point) on the Pong stand-in ROM with the paper's
Pong spec, frame skip 4, uniform random actions from the
device generator.  One "step" = one octax_step launch over all envs.  The
smaller configs are reported in the "sweep" key and are parity-test cases.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU)
"""
from __future__ import annotations

import argparse
import json
import os
import re
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "env steps/sec (and frames/sec) at 1/2/4/8 B200 vs #parallel envs"
PAPER_CONTEXT = {"value": 350000, "unit": "env steps/s", "envs": 8192,
                 "hardware": "RTX 3090", "source": "P:51, P:228-231 (context, not this workload)"}

# algorithmic HBM bytes per env step: history planes read
# 768 + new ring plane 256 + obs 1024 + VM state read+write 2*(16+16+16+8) + stack
# read 32 (+ write 32 only after CALL, not counted) + action 4 + reward 4 + done 1
ALG_BYTES_PER_ENV_STEP = 768 + 256 + 1024 + 2 * (16 + 16 + 16 + 8) + 32 + 4 + 4 + 1


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max(float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[2 + k].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------ CPU oracle (baseline / reference arm)
def _oracle_worker(game, obs_format, envs_per_proc, steps, rounds, k, barrier, q):
    import numpy as np

    import oracle
    import workloads
    rom, spec = workloads.game(game, obs_format=obs_format)
    na = workloads.n_actions(spec)
    off = k * envs_per_proc
    e = oracle.OracleEnv(rom, spec, envs_per_proc, workloads.ENV_SEED, off)
    # the same Philox domain-1 action stream the GPU arm draws on the device (octax_gen_actions),
    # for the same global ids, generated before the timed rounds
    acts = [np.ascontiguousarray(oracle.synthetic_actions(workloads.ACTION_SEED, t, range(off, off + envs_per_proc), na))
            for t in range(steps)]
    obs = np.zeros((envs_per_proc, e.obs_per_env), np.uint8)
    rew = np.zeros(envs_per_proc, np.float32)
    done = np.zeros(envs_per_proc, np.uint8)
    for r in range(rounds):
        barrier.wait()
        t0 = time.perf_counter()
        for t in range(steps):
            e.step_into(acts[t], obs, rew, done)
        q.put((r, time.perf_counter() - t0))


def oracle_throughput(game: str, envs_per_proc: int, steps: int, procs: int | None = None, rounds: int = 1,
                      obs_format: int = 0):
    """The oracle as it stands, on the host cores: C worker processes, each its
    own single-threaded oracle instance over a disjoint env range, started
    together for each round.  Returns (per-round aggregate steps/s list, cores,
    sample description)."""
    import multiprocessing as mp
    C = procs or len(os.sched_getaffinity(0))
    ctx = mp.get_context("spawn")
    barrier, q = ctx.Barrier(C), ctx.Queue()
    ps = [ctx.Process(target=_oracle_worker, args=(game, obs_format, envs_per_proc, steps, rounds, k, barrier, q))
          for k in range(C)]
    for p in ps:
        p.start()
    worst = [0.0] * rounds
    for _ in range(C * rounds):
        r, t = q.get()
        worst[r] = max(worst[r], t)
    for p in ps:
        p.join()
    total = C * envs_per_proc * steps
    cpu = ""
    try:
        with open("/proc/cpuinfo") as f:
            cpu = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except Exception:
        pass
    sample = (f"{game}: {C} processes x {envs_per_proc} envs x {steps} steps = {total} env steps per round, "
              f"{'bool' if obs_format & 1 else 'packed'} obs, Philox domain-1 actions of global ids "
              f"0..{C * envs_per_proc - 1}, slowest process {sorted(worst)[len(worst) // 2]:.2f} s (median round); {cpu}")
    return [total / w for w in worst], C, sample


ACTIONS = "uniform random, Philox4x32-10 domain-1 stream keyed by global env id (SURVEY App. C)"


def arm_config(args, spec, n, world, impl="ours", sample=None):
    """The bench line's `config`.  Both arms share the workload identity keys (game, spec,
    obs format, actions, the per-GPU env count the line stands for); each states what it
    actually ran: ours the device path over all n envs per GPU, the reference arm (the CPU
    oracle) a bounded sample of the same workload (`sample`)."""
    c = {"workload": f"BASELINE configs[4] per-GPU slice: {args.game} (labelled stand-in ROM, "
                     f"paper Pong spec P:152/P:156), {n} envs per GPU, frame_skip 4, ipf 12, "
                     f"{'bool [n,4,64,32]' if args.obs == 'bool' else 'packed 4-plane'} obs",
         "game": args.game, "envs_per_gpu": n, "global_envs": world * n,
         "frame_skip": spec["frame_skip"], "instructions_per_frame": spec["instructions_per_frame"],
         "obs_format": "packed [n,4,32,8]" if args.obs == "packed" else "bool [n,4,64,32] (x-major, P:146)",
         "actions": ACTIONS, "parallelism": f"env-sharded x{world}"}
    if impl == "ours":
        c["ran"] = (f"device: {n} envs per GPU x {world} GPU(s), actions generated on the device "
                    "(octax_gen_actions) before the timed region")
        c["l2"] = (f"inputs larger than L2: ~{ALG_BYTES_PER_ENV_STEP * n / 2**30:.2f} GiB touched per step "
                   "vs 126 MB L2 (no flush needed)")
    else:
        c["ran"] = ("host CPU oracle (oracle/octax_oracle.c, single-threaded C, one process per core): "
                    f"a bounded sample of this workload, {sample['envs']} envs x {sample['steps']} steps per "
                    "round, actions from the oracle's own Philox (oracle.synthetic_actions) for the same "
                    "global ids, generated before the timed rounds")
        c["sample"] = sample
    return c


def run_reference(args):
    """--impl reference: the oracle (this tier's reference arm) on the host cores,
    same game / metric / unit as our arm; each step = one bounded sample round."""
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    envs_per_proc, steps_per_round = 256, 25
    import workloads
    _, spec = workloads.game(args.game, obs_format=1 if args.obs == "bool" else 0)
    fmt = 1 if args.obs == "bool" else 0
    vals, C, sample = oracle_throughput(args.game, envs_per_proc, steps_per_round,
                                        procs=args.cpu_procs, rounds=args.warmup + args.steps, obs_format=fmt)
    timed = sorted(vals[args.warmup:])
    v = timed[len(timed) // 2]
    out = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "env steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": C * envs_per_proc * steps_per_round / v * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": arm_config(args, spec, args.envs, _env_int("WORLD_SIZE", 1), impl="reference",
                             sample={"processes": C, "envs_per_process": envs_per_proc, "envs": C * envs_per_proc,
                                     "steps": steps_per_round, "obs_format": fmt}),
        "cpu_baseline": {"value": v, "unit": "env steps/s", "cores": C, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "env steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "frames_per_s": 4 * v,
    }
    print(json.dumps(out), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
def time_config(rom, spec, n, steps, warmup, rank_offset, aseed, torch, OctaxEnv, barrier=None,
                keep=False, graph=False, rollout=0, on_rollout=None, kernel=None):
    """Time `steps` octax_step launches (each = one step of all n envs) on a dedicated
    stream with CUDA events; graph=True captures the K launches in one CUDA graph
    (K % 4 == 0 keeps the 4-slot display ring aligned across replays).  on_rollout(env, stream)
    runs inside the timed region after every `rollout` steps and after the last one (the
    per-rollout statistics all-reduce of SURVEY §8(e))."""
    stream = torch.cuda.Stream()
    env = OctaxEnv(rom, spec, n, 0x0C7A251001764000, env_offset=rank_offset, stream=stream, kernel=kernel)
    T = warmup + steps
    acts = torch.empty((T, n), dtype=torch.int32, device="cuda")
    with torch.cuda.stream(stream):
        for t in range(T):
            env.gen_actions(aseed, t, acts[t])
    obs, rew, done = env.obs, env.reward, env.done
    for t in range(warmup):
        env.step_into(acts[t], obs, rew, done)
    g = None
    if graph:
        assert steps % 4 == 0
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for k in range(steps):
                env.step_into(acts[warmup + k], obs, rew, done)
        with torch.cuda.stream(stream):
            g.replay()  # warm replay
    torch.cuda.synchronize()
    if barrier:
        barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record(stream)
    if graph:
        with torch.cuda.stream(stream):
            g.replay()
        ev[steps].record(stream)
    else:
        for k in range(steps):
            env.step_into(acts[warmup + k], obs, rew, done)
            if on_rollout is not None and ((rollout and (k + 1) % rollout == 0) or k == steps - 1):
                on_rollout(env, stream)
            ev[k + 1].record(stream)
    torch.cuda.synchronize()
    if barrier:
        barrier()
    per = [] if graph else [ev[k].elapsed_time(ev[k + 1]) for k in range(steps)]
    total_ms = ev[0].elapsed_time(ev[steps])
    if not keep:
        del g, acts
        env.close()
        return total_ms, per, None
    return total_ms, per, (env, acts, stream)


def time_rollout(rom, spec, n, T, reps, warmup_reps, rank_offset, aseed, torch, OctaxEnv, barrier=None,
                 on_rollout=None, with_obs=True, kernel=None):
    """Fused rollout mode (octax_rollout, SURVEY d.8 mode "fused"): `reps` launches of T steps
    each, actions generated inside the kernel (the step mode's actions are generated before its
    timed region, so this mode does strictly more work per step), obs / reward / done written
    every step into the same [n] buffers as the step mode.  CUDA events on the env's stream;
    on_rollout(env, stream) after every rollout inside the timed region.  Returns
    (total_ms, per-rollout ms, env)."""
    stream = torch.cuda.Stream()
    env = OctaxEnv(rom, spec, n, 0x0C7A251001764000, env_offset=rank_offset, stream=stream, kernel=kernel)
    obs, rew, done = env.obs if with_obs else None, env.reward, env.done
    t = 0
    with torch.cuda.stream(stream):
        for _ in range(warmup_reps):
            env.rollout_into(T, obs, rew, done, aseed=aseed, t0=t)
            t += T
    torch.cuda.synchronize()
    if barrier:
        barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record(stream)
    with torch.cuda.stream(stream):
        for k in range(reps):
            env.rollout_into(T, obs, rew, done, aseed=aseed, t0=t)
            t += T
            if on_rollout is not None:
                on_rollout(env, stream)
            ev[k + 1].record(stream)
    torch.cuda.synchronize()
    if barrier:
        barrier()
    per = [ev[k].elapsed_time(ev[k + 1]) for k in range(reps)]
    return ev[0].elapsed_time(ev[reps]), per, env


def fused_model(game, n):
    """ncu counts of one fused rollout launch (profiles/latest_fused_full.json, per env step) if
    the capture is of this build (device-code digest), game and env count."""
    try:
        with open(os.path.join(ROOT, "profiles", "latest_fused_full.json")) as f:
            j = json.load(f)
        from paper_2510_01764_b200 import octax
        from paper_2510_01764_b200.build import device_code_digest
        if (j.get("sass_sha256") == device_code_digest(octax.SO_PATH) and j.get("game") == game
                and "octax_kernel<2," in str(j.get("kernel_symbol", "")) and j.get("envs_per_launch") == n):
            return j
    except Exception:
        pass
    return None


def issue_model(game, n):
    """ncu instruction counts of the step kernel (profiles/latest_step_full.json), used for the
    ALU-pipe and issue roofs only if the profile is of THIS build and workload: the device-code
    digest (cuobjdump -sass sha256) of the loaded library, the step-kernel symbol, the game and
    the env count must all match.  Returns (counts or None, reason)."""
    try:
        with open(os.path.join(ROOT, "profiles", "latest_step_full.json")) as f:
            j = json.load(f)
    except Exception as ex:
        return None, f"no profile: {ex}"
    from paper_2510_01764_b200 import octax
    from paper_2510_01764_b200.build import device_code_digest
    have = device_code_digest(octax.SO_PATH)
    why = []
    if j.get("sass_sha256") is None or j.get("sass_sha256") != have:
        why.append(f"device code {str(j.get('sass_sha256'))[:12]} != loaded {str(have)[:12]}")
    if not re.search(r"octax_kernel<(\(int\))?0,", str(j.get("kernel_symbol", ""))):
        why.append("profile is not of the step kernel")
    if j.get("game") != game:
        why.append(f"game {j.get('game')} != {game}")
    if j.get("envs") != n:
        why.append(f"envs {j.get('envs')} != {n}")
    if why:
        return None, "stale ncu profile: " + "; ".join(why)
    return j, "profiles/latest_step_full.json (same device code, kernel, game and env count)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--envs", type=int, default=1 << 20, help="envs per GPU")
    ap.add_argument("--game", default="pong_standin")
    ap.add_argument("--obs", default="packed", choices=["packed", "bool"],
                    help="observation layout (bool = the paper's dense x-major [n,4,64,32])")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fused", action="store_true", help="skip the fused-rollout-mode measurement")
    ap.add_argument("--no-fused-noobs", action="store_true", help="skip the observation-less fused rollouts")
    ap.add_argument("--dist-backend", default="auto", choices=["auto", "nccl", "gloo"],
                    help="auto: nccl with one GPU per rank; gloo when ranks share a device "
                         "(a functional multi-rank run on fewer GPUs than ranks)")
    ap.add_argument("--rollout", type=int, default=100,
                    help="steps per rollout: one int64[4] statistics all-reduce per rollout, inside "
                         "the timed region (P:228 100-step rollouts, SURVEY §8(e))")
    ap.add_argument("--max-episode-steps", type=int, default=None,
                    help="override the game spec's truncation length (tests: force auto-resets)")
    ap.add_argument("--cpu-procs", type=int, default=None,
                    help="--impl reference: oracle processes (default: one per host core)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import workloads
    from paper_2510_01764_b200 import OctaxEnv

    from paper_2510_01764_b200 import dist as odist
    rank, world, local = odist.rank_info()
    ndev = torch.cuda.device_count()
    dev = local % ndev
    torch.cuda.set_device(dev)
    backend = args.dist_backend
    if backend == "auto":
        backend = "nccl" if world <= ndev else "gloo"
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")

    def barrier():
        if world > 1:
            dist.barrier()

    rom, spec = workloads.game(args.game, obs_format=1 if args.obs == "bool" else 0)
    if args.max_episode_steps is not None:
        spec = dict(spec, max_episode_steps=args.max_episode_steps)
    n = args.envs
    offset, _ = odist.shard(rank, world, n)

    # ---- headline: n envs per GPU, K timed steps; after every rollout (and the last step) the
    #      int64[4] episode statistics are all-reduced inside the timed region
    st = torch.zeros(4, dtype=torch.int64, device="cuda")
    n_reduce = [0]

    def on_rollout(env, stream):
        with torch.cuda.stream(stream):
            env.stats_device(st)
            odist.reduce_stats(st)
        n_reduce[0] += 1

    with ClockSampler(dev) as clk:
        total_ms, per, kept = time_config(rom, spec, n, args.steps, args.warmup, offset,
                                          workloads.ACTION_SEED, torch, OctaxEnv, barrier, keep=True,
                                          rollout=args.rollout, on_rollout=on_rollout)
        env, acts, stream = kept
        stream.synchronize()
    # per-env 64-bit state digests after the timed steps (SURVEY d.1 item 4): rank 0's shard
    # sum is the same for every N (trajectories are keyed by global id), the all-rank sum
    # covers every env of the job (int64 all-reduce = sum mod 2^64)
    _, dsum = env.state_digests()
    dall = torch.tensor([dsum - (1 << 64) if dsum >= (1 << 63) else dsum], dtype=torch.int64, device="cuda")
    odist.reduce_stats(dall)
    digest = {"rank0_shard_sum": f"{dsum:016x}" if rank == 0 else None,
              "all_ranks_sum": f"{int(dall.item()) % (1 << 64):016x}", "envs": world * n,
              "def": "sum mod 2^64 of FNV-1a-64 of each env's canonical state (octax_state_digests)"}
    t_ms = odist.max_over_ranks(torch.tensor([total_ms], dtype=torch.float64, device="cuda"))
    t_max = float(t_ms.item())
    value = world * n * args.steps / (t_max / 1e3)
    kernel_ms = sorted(per)[len(per) // 2]

    hbm_peak, peak_src = _peaks()
    achieved = ALG_BYTES_PER_ENV_STEP * n / (kernel_ms / 1e3) / 1e9
    traffic = None

    # ALU-pipe roof (the binding one): 148 SMs x 4 SMSPs x one
    # ALU-pipe warp instruction per 2 cycles (B300_MICROARCH: alu pipe rt_SMSP = 2) x 32
    # lanes x the SM clock sampled during the timed region; the work per env step is the
    # kernel's ALU-pipe instruction count measured by ncu (profiles/latest_step_full.json).
    alu = None
    im, im_why = issue_model(args.game, n)
    clk_mhz = None
    try:
        clk_mhz = clk.summary()["sm_mhz"]
    except Exception:
        pass
    f_sm = (clk_mhz or 1965.0) * 1e6
    if im and im.get("dram_bytes_per_launch"):
        traffic = im["dram_bytes_per_launch"]   # ncu --set full of this build, same launch configuration
    if im and im.get("alu_warp_instr_per_env_step"):
        peak_alu = 148 * 4 * 0.5 * 32 * f_sm / 1e9          # G thread-ALU-ops / s
        ach_alu = im["alu_warp_instr_per_env_step"] * 32 * value / world / 1e9
        alu = {"achieved": ach_alu, "peak": peak_alu, "unit": "G ALU-pipe thread-instr/s",
               "frac": ach_alu / peak_alu, "alu_warp_instr_per_env_step": im["alu_warp_instr_per_env_step"],
               "all_warp_instr_per_env_step": im.get("warp_instr_per_env_step"),
               "warp_exec_efficiency": im.get("warp_exec_efficiency"),
               "ncu_alu_pipe_pct_of_peak": im.get("alu_pipe_pct_of_peak"),
               "sm_mhz": f_sm / 1e6, "source": im.get("source"), "provenance": im_why,
               "sass_sha256": im.get("sass_sha256")}

    # issue roof (SURVEY d.2): 148 SMs x 4 schedulers x 1 warp instruction per cycle x f_SM,
    # against all warp instructions per env step measured by ncu (same source as the ALU count)
    # SURVEY d.2's a-priori issue roof (I_step ~ 2,000 thread instructions per env step, estimated
    # before any kernel existed): context for the self-referential measured-instruction roofs
    survey_issue = {"I_step_thread_estimate": 2000, "roof_env_steps_per_s": 148 * 4 * 32 * f_sm / 2000,
                    "frac": value / world / (148 * 4 * 32 * f_sm / 2000),
                    "I_step_thread_measured": (im["warp_instr_per_env_step"] * 32 * im.get("warp_exec_efficiency", 1.0)
                                               if im and im.get("warp_instr_per_env_step") else None)}
    issue = None
    if im and im.get("warp_instr_per_env_step"):
        peak_iss = 148 * 4 * f_sm / 1e9
        ach_iss = im["warp_instr_per_env_step"] * value / world / 1e9
        issue = {"achieved": ach_iss, "peak": peak_iss, "unit": "G warp-instr/s", "frac": ach_iss / peak_iss,
                 "warp_instr_per_env_step": im["warp_instr_per_env_step"]}

    # ---- e2e through the host-buffer C-ABI calls (H2D actions, D2H results, from / to pinned
    #      host memory, every step inside the timed region).  Headline: octax_step_host_frame,
    #      which ships the newest display + reward + done (the host keeps the 3 older displays,
    #      include/octax.h); "full_obs": octax_step_host shipping the whole 4-plane stack.
    e2e = None
    if not args.no_e2e:
        K = max(3, min(args.steps, 10))
        a_h = torch.empty((K, n), dtype=torch.int32).pin_memory()
        a_h.copy_(acts[:K].cpu())
        o_h = torch.empty((n, env.obs_per_env), dtype=torch.uint8).pin_memory()
        f_h = torch.empty((n, 32, 8), dtype=torch.uint8).pin_memory()
        r_h = torch.empty(n, dtype=torch.float32).pin_memory()
        d_h = torch.empty(n, dtype=torch.uint8).pin_memory()
        nd = lambda t: t.numpy()

        def run(fn, out):
            fn(nd(a_h[0]), nd(out), nd(r_h), nd(d_h))  # warm the staging buffers
            barrier()
            t0 = time.perf_counter()
            for k in range(K):
                fn(nd(a_h[k]), nd(out), nd(r_h), nd(d_h))
            dt = odist.max_over_ranks(torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda"))
            return world * n * K / float(dt.item())

        # the link roof: this box's pinned D2H copy bandwidth (plain cudaMemcpyAsync of a device
        # buffer into the pinned obs buffer, best of 3)
        src = torch.empty((n, env.obs_per_env), dtype=torch.uint8, device="cuda")
        best = None
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            o_h.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            t = time.perf_counter() - t0
            best = t if best is None else min(best, t)
        d2h_gbs = o_h.numel() / best / 1e9
        del src

        def link(value, bytes_step):
            roof = d2h_gbs * 1e9 / (bytes_step / n) * world
            return {"d2h_gbs_measured": d2h_gbs, "bytes_per_env_step": bytes_step / n,
                    "roof_env_steps_per_s": roof, "frac": value / roof}

        vf = run(env.step_host_frame, f_h)
        vfull = run(env.step_host, o_h)
        bf, bfull = (4 + 256 + 4 + 1) * n, (4 + env.obs_per_env + 4 + 1) * n
        e2e = {"value": vf, "unit": "env steps/s", "h2d_bytes_per_step": 4 * n,
               "d2h_bytes_per_step": (256 + 4 + 1) * n, "steps": K,
               "path": "octax_step_host_frame (pinned host buffers; newest display + reward + done, "
                       "the host keeps the three older displays)",
               "link": link(vf, bf),
               "full_obs": {"value": vfull, "h2d_bytes_per_step": 4 * n,
                            "d2h_bytes_per_step": (env.obs_per_env + 4 + 1) * n,
                            "path": "octax_step_host (whole 4-plane stack)", "link": link(vfull, bfull)}}
    env.close()
    del acts
    torch.cuda.empty_cache()

    # ---- fused rollout mode at the headline size (SURVEY d.8 mode "fused"): 100-step rollouts
    #       in one launch each, in-kernel actions, one stats all-reduce per rollout
    fused = None
    if not args.no_fused:
        fst = torch.zeros(4, dtype=torch.int64, device="cuda")

        def on_fused(env_, stream_):
            with torch.cuda.stream(stream_):
                env_.stats_device(fst)
                odist.reduce_stats(fst)

        R = 2
        tm, per_r, fenv = time_rollout(rom, spec, n, 100, R, 1, offset, workloads.ACTION_SEED, torch, OctaxEnv,
                                       barrier, on_rollout=on_fused)
        fenv.close()
        tf = float(odist.max_over_ranks(torch.tensor([tm], dtype=torch.float64, device="cuda")).item())
        fv = world * n * 100 * R / (tf / 1e3)
        # its rooflines: HBM with the fused mode's 1,797 algorithmic B per env step (no state round
        # trip, no framebuffer TMA read, in-kernel actions), ALU pipe with the step
        # kernel's measured instruction count (the same interpreter; an upper bound)
        f_bytes = 512 + 1024 + 256 + 4 + 1
        hbm_f = f_bytes * fv / world / 1e9
        fused_roof = {"hbm": {"achieved": hbm_f, "peak": hbm_peak, "unit": "GB/s", "frac": hbm_f / hbm_peak,
                              "alg_bytes_per_env_step": f_bytes}}
        fm = fused_model(args.game, n)
        if fm and fm.get("alu_warp_instr_per_env_step"):
            a_f = fm["alu_warp_instr_per_env_step"] * 32 * fv / world / 1e9
            peak_alu = 148 * 4 * 0.5 * 32 * f_sm / 1e9
            fused_roof["alu"] = {"achieved": a_f, "peak": peak_alu, "frac": a_f / peak_alu,
                                 "alu_warp_instr_per_env_step": fm["alu_warp_instr_per_env_step"],
                                 "source": "profiles/latest_fused_full.json (ncu of one rollout launch of this build)"}
        elif alu:
            a_f = alu["alu_warp_instr_per_env_step"] * 32 * fv / world / 1e9
            fused_roof["alu"] = {"achieved": a_f, "peak": alu["peak"], "frac": a_f / alu["peak"],
                                 "note": "step kernel's ALU-pipe instructions per env step (no fused capture of this build)"}
        fused = {"mode": "fused", "steps_per_rollout": 100, "rollouts_timed": R, "warmup_rollouts": 1,
                 "steps_per_s": fv, "frames_per_s": 4 * fv, "ms_per_step": tf / (100 * R), "roofline": fused_roof,
                 "ms_per_rollout_median": sorted(per_r)[len(per_r) // 2],
                 "vs_step_mode": fv / value, "stats": [int(x) for x in fst.cpu().tolist()],
                 "actions": "generated inside the rollout kernel (Philox domain 1, same stream as octax_gen_actions)",
                 "no_obs": None,
                 "outputs": ("obs / reward / done written every step (same [n] buffers as the step mode)"
                             if args.obs == "packed" else
                             "packed obs / reward / done written every step; the bool [n,4,64,32] expansion runs "
                             "once, for the last step (stride 0: every step overwrites the same buffer, so the "
                             "earlier steps' bool obs are never observable)")}
        # the same rollouts without observations (octax_rollout obs_out = NULL: rewards / dones
        # only, e.g. policy-free evaluation) -- the interpreter with no obs I/O, context only
        if not args.no_fused_noobs:
            tm, _, fenv = time_rollout(rom, spec, n, 100, R, 1, offset, workloads.ACTION_SEED, torch, OctaxEnv,
                                       barrier, with_obs=False)
            fenv.close()
            tn = float(odist.max_over_ranks(torch.tensor([tm], dtype=torch.float64, device="cuda")).item())
            fused["no_obs"] = {"steps_per_s": world * n * 100 * R / (tn / 1e3), "ms_per_step": tn / (100 * R),
                               "note": "octax_rollout with obs_out = NULL (rewards / dones only): not the "
                                       "headline workload"}
        torch.cuda.empty_cache()

    # ---- sweep of smaller per-GPU env counts (context; parity-test configs): per-launch
    #      and CUDA-graph-captured (launch overhead dominates below ~64K envs)
    sweep = []
    if not args.no_sweep:
        ks = max(4, (args.steps // 4) * 4)
        for m in (1024, 4096, 65536, 262144):
            if m >= n:
                continue
            row = {"envs_per_gpu": m}
            for graph in (False, True):
                tm, _, _ = time_config(rom, spec, m, ks, args.warmup, odist.shard(rank, world, m)[0],
                                       workloads.ACTION_SEED, torch, OctaxEnv, barrier, graph=graph)
                tt = float(odist.max_over_ranks(torch.tensor([tm], dtype=torch.float64, device="cuda")).item())
                sps = world * m * ks / (tt / 1e3)
                key = "graph" if graph else "launch"
                row[f"steps_per_s_{key}"] = sps
                row[f"ms_per_step_{key}"] = tt / ks
            row["frames_per_s_graph"] = 4 * row["steps_per_s_graph"]
            tm, _, fenv = time_rollout(rom, spec, m, 100, 2, 1, odist.shard(rank, world, m)[0],
                                       workloads.ACTION_SEED, torch, OctaxEnv, barrier)
            row["kernel"] = fenv.kernel  # OCTAX_KERNEL_AUTO's choice for this batch size
            fenv.close()
            tt = float(odist.max_over_ranks(torch.tensor([tm], dtype=torch.float64, device="cuda")).item())
            row["steps_per_s_fused"] = world * m * 200 / (tt / 1e3)
            row["ms_per_step_fused"] = tt / 200
            if row["kernel"] == "warp":  # the lane-per-env kernel on the same batch, for comparison
                lk = {}
                tm, _, _ = time_config(rom, spec, m, ks, args.warmup, odist.shard(rank, world, m)[0],
                                       workloads.ACTION_SEED, torch, OctaxEnv, barrier, kernel="lane")
                tt = float(odist.max_over_ranks(torch.tensor([tm], dtype=torch.float64, device="cuda")).item())
                lk["steps_per_s_launch"] = world * m * ks / (tt / 1e3)
                tm, _, fenv = time_rollout(rom, spec, m, 100, 2, 1, odist.shard(rank, world, m)[0],
                                           workloads.ACTION_SEED, torch, OctaxEnv, barrier, kernel="lane")
                fenv.close()
                tt = float(odist.max_over_ranks(torch.tensor([tm], dtype=torch.float64, device="cuda")).item())
                lk["steps_per_s_fused"] = world * m * 200 / (tt / 1e3)
                row["lane_kernel"] = lk
            sweep.append(row)
        sweep.append({"envs_per_gpu": n, "kernel": "lane" if n > int(os.environ.get("OCTAX_WARP_AUTO_MAX", 4096)) else "warp",
                      "steps_per_s_launch": value, "frames_per_s_launch": 4 * value,
                      "ms_per_step_launch": t_max / args.steps,
                      **({"steps_per_s_fused": fused["steps_per_s"], "ms_per_step_fused": fused["ms_per_step"]}
                         if fused else {})})

    # ---- many small handles at once (context): the paper's scale is thousands of envs per game,
    #      which leaves most of a B200 idle -- 16 handles of 4,096 envs (the five workloads in turn),
    #      each on its own stream, run 100-step fused rollouts concurrently; aggregate env steps/s
    concurrent = None
    if not args.no_sweep and not args.no_fused:
        names = ["pong_standin", "brix_standin", "target_shooter_level1", "target_shooter_level2",
                 "target_shooter_level3"]
        rates = {}
        # AUTO gives each 4,096-env handle the warp-per-env kernel (best for ONE such handle); 16
        # of them together fill the GPU, where the lane-per-env kernel's throughput wins
        for kern in ("lane", "warp"):
            hs = []
            for k in range(16):
                grom, gspec = workloads.game(names[k % len(names)])
                st_k = torch.cuda.Stream()
                e_k = OctaxEnv(grom, gspec, 4096, 0x0C7A251001764000, env_offset=odist.shard(rank, world, 4096 * 16)[0]
                               + 4096 * k, stream=st_k, kernel=kern)
                hs.append((e_k, st_k))
            for rep in range(2):  # warm-up rollout, then the timed one
                torch.cuda.synchronize()
                barrier()
                start = torch.cuda.Event(enable_timing=True)
                start.record()
                ends = []
                for e_k, st_k in hs:
                    st_k.wait_event(start)
                    with torch.cuda.stream(st_k):
                        e_k.rollout_into(100, e_k.obs, e_k.reward, e_k.done, aseed=workloads.ACTION_SEED, t0=100 * rep)
                    end = torch.cuda.Event(enable_timing=True)
                    end.record(st_k)
                    ends.append(end)
                torch.cuda.synchronize()
                dt = max(start.elapsed_time(end) for end in ends) / 1e3  # CUDA events: first launch to last end
            dt = float(odist.max_over_ranks(torch.tensor([dt], dtype=torch.float64, device="cuda")).item())
            rates[kern] = world * 16 * 4096 * 100 / dt
            for e_k, _ in hs:
                e_k.close()
            torch.cuda.empty_cache()
        concurrent = {"handles": 16, "envs_per_handle": 4096, "steps": 100, "mode": "fused", "kernel": "lane",
                      "steps_per_s": rates["lane"], "warp_kernel_steps_per_s": rates["warp"],
                      "single_handle_steps_per_s": next((r.get("steps_per_s_fused") for r in sweep
                                                         if r.get("envs_per_gpu") == 4096), None),
                      "note": "octax_set_kernel(LANE) on every handle: AUTO picks per handle (warp for one "
                              "4,096-env handle); concurrent handles that together fill the GPU run faster on "
                              "the lane-per-env kernel",
                      "timing": "CUDA events: a start event all 16 streams wait on, to the latest of their end events"}

    # ---- per-game throughput at BASELINE configs[3]'s size (262,144 envs per GPU): the
    #      paper claims one number for all games; a SIMT interpreter is game dependent
    games = []
    if not args.no_sweep:
        m = min(n, 262144)
        for g in ("pong_standin", "brix_standin", "target_shooter_level1", "target_shooter_level2",
                  "target_shooter_level3"):
            grom, gspec = workloads.game(g)
            tm, _, _ = time_config(grom, gspec, m, args.steps, args.warmup, odist.shard(rank, world, m)[0],
                                   workloads.ACTION_SEED, torch, OctaxEnv, barrier)
            tt = float(odist.max_over_ranks(torch.tensor([tm], dtype=torch.float64, device="cuda")).item())
            sps = world * m * args.steps / (tt / 1e3)
            row = {"game": g, "envs_per_gpu": m, "steps_per_s": sps, "frames_per_s": 4 * sps,
                   "source": "paper listing (App. D)" if g.startswith("target") else "labelled stand-in"}
            if not args.no_fused:  # the same workload as 100-step fused rollouts
                tm, _, fenv = time_rollout(grom, gspec, m, 100, 2, 1, odist.shard(rank, world, m)[0],
                                           workloads.ACTION_SEED, torch, OctaxEnv, barrier)
                fenv.close()
                tt = float(odist.max_over_ranks(torch.tensor([tm], dtype=torch.float64, device="cuda")).item())
                row["steps_per_s_fused"] = world * m * 200 / (tt / 1e3)
            games.append(row)

    # the oracle on the host cores, rank 0 only, after every rank's GPU work (the other ranks
    # wait at the closing barrier)
    cpu = None
    if rank == 0 and not args.no_cpu:
        vals, C, sample = oracle_throughput(args.game, 256, 400, obs_format=1 if args.obs == "bool" else 0)
        v = vals[0]
        cpu = {"value": v, "unit": "env steps/s", "cores": C, "kind": "oracle", "sample": sample}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "env steps/s",
            "frames_per_s": 4 * value,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": arm_config(args, spec, n, world),
            "dist": {"backend": backend if world > 1 else None, "world": world, "devices": ndev,
                     "stats_allreduces_in_timed_region": n_reduce[0], "rollout_steps": args.rollout,
                     "note": ("ranks share a device: functional multi-rank run, not a scaling number"
                              if world > ndev else "one GPU per rank")},
            "roofline": ({"bound": "alu", "achieved": alu["achieved"], "peak": alu["peak"], "unit": alu["unit"],
                          "frac": alu["frac"], "traffic": traffic, "kernel": "octax_kernel<MODE_STEP>",
                          "kernel_ms_median": kernel_ms, "alu": alu, "issue": issue, "issue_survey_estimate": survey_issue,
                          "hbm": {"achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                                  "alg_bytes_per_env_step": ALG_BYTES_PER_ENV_STEP, "peak_source": peak_src,
                                  "roof_env_steps_per_s": hbm_peak * 1e9 / ALG_BYTES_PER_ENV_STEP}}
                         if alu else
                         {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                          "frac": achieved / hbm_peak, "traffic": traffic, "kernel": "octax_kernel<MODE_STEP>",
                          "alu": None, "alu_unavailable": im_why,
                          "kernel_ms_median": kernel_ms, "alg_bytes_per_env_step": ALG_BYTES_PER_ENV_STEP,
                          "peak_source": peak_src}),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "fused": fused,
            "state_digest": digest,
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
            "stats": [int(x) for x in st.cpu().tolist()],
            "sweep": sweep,
            "games": games,
            "concurrent_handles": concurrent,
            "paper_context": PAPER_CONTEXT,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
