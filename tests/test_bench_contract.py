"""bench.py's reference arm (the CPU oracle, this tier's reference implementation) runs on
the host: its JSON line must carry the driver contract's keys, and under torchrun only rank
0 prints (the other ranks exit 0 without work)."""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env=None):
    env = dict(os.environ, **(extra_env or {}))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0", "--cpu-procs", "2"],
                       capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout


def test_reference_arm_json_line():
    lines = [l for l in _run().splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "env steps/s"
    assert d["higher_is_better"] is True and d["steps"] == 1 and d["warmup"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == 2 and cb["value"] == d["value"] and cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0
    # the workload identity keys of our arm's `config` (bench.arm_config), so the driver compares
    # like with like, plus what this arm actually ran: a bounded oracle sample
    c = d["config"]
    assert c["game"] == "pong_standin" and c["envs_per_gpu"] == 1048576 and c["global_envs"] == 1048576
    assert c["frame_skip"] == 4 and c["instructions_per_frame"] == 12 and c["workload"].startswith("BASELINE configs[4]")
    assert "device" not in c["workload"] and "Philox" in c["actions"]
    assert c["sample"]["processes"] == 2 and c["sample"]["envs"] == 2 * c["sample"]["envs_per_process"]
    assert "oracle" in c["ran"] and str(c["sample"]["envs"]) in c["ran"]
    import argparse
    sys.path.insert(0, ROOT)
    import bench
    import workloads
    _, spec = workloads.game("pong_standin")
    ours = bench.arm_config(argparse.Namespace(game="pong_standin", obs="packed"), spec, 1048576, 1)
    shared = ("workload", "game", "envs_per_gpu", "global_envs", "frame_skip", "instructions_per_frame",
              "obs_format", "actions", "parallelism")
    assert {k: ours[k] for k in shared} == {k: c[k] for k in shared}
    assert "device" in ours["ran"] and "sample" not in ours


def test_reference_arm_bool_obs_runs_bool_oracle():
    env = dict(os.environ)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--obs", "bool",
                        "--steps", "1", "--warmup", "0", "--cpu-procs", "1"],
                       capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["config"]["sample"]["obs_format"] == 1 and "bool obs" in d["cpu_baseline"]["sample"]


def test_reference_arm_nonzero_rank_is_silent():
    assert _run({"RANK": "1", "WORLD_SIZE": "2"}).strip() == ""
