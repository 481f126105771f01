#!/usr/bin/env python
"""Copy one evidence pass (`scripts/gpu_r2_full.sh` + `scripts/gpu_r2_misc.sh`, results merged into
gpurun_out/) into profiles/ under a kernel version tag, refresh the digest-stamped
latest_step_full.json / latest_fused_full.json that bench.py reads, and regenerate the derived
tables (SURVEY d.4 ncu table, per-region source attribution, launch list).

    python scripts/collect_evidence.py r02_v40

Refuses to run when the captures' device-code digest differs from the in-tree library's (the
evidence would not describe the code that `bench.py` loads)."""
from __future__ import annotations

import glob
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def main():
    tag = sys.argv[1]
    from paper_2510_01764_b200.build import SO, device_code_digest
    have = device_code_digest(SO)
    step = json.load(open(os.path.join(G, "step_full_1048576.json")))
    if step.get("sass_sha256") != have:
        sys.exit(f"capture digest {str(step.get('sass_sha256'))[:16]} != in-tree library {str(have)[:16]}")
    caps = []
    for f in sorted(glob.glob(os.path.join(G, "step_full_*.json"))):
        j = json.load(open(f))
        if j.get("sass_sha256") != have:
            continue
        name = os.path.basename(f)[len("step_"):]
        shutil.copy(f, os.path.join(P, f"{tag}_{name}"))
        caps.append(os.path.join(P, f"{tag}_{name}"))
    shutil.copy(os.path.join(P, f"{tag}_full_1048576.json"), os.path.join(P, "latest_step_full.json"))
    fz = os.path.join(G, "fused_full_1048576.json")
    if os.path.exists(fz):
        j = json.load(open(fz))
        if j.get("sass_sha256") == have:
            j["envs_per_launch"] = 1048576
            for out in (f"{tag}_fused_full_1048576.json", "latest_fused_full.json"):
                json.dump(j, open(os.path.join(P, out), "w"), indent=1)
    for f in sorted(glob.glob(os.path.join(G, "warp_full_*.json"))):  # warp-per-env kernel captures
        if json.load(open(f)).get("sass_sha256") == have:
            shutil.copy(f, os.path.join(P, f"{tag}_{os.path.basename(f)}"))
            caps.append(os.path.join(P, f"{tag}_{os.path.basename(f)}"))
    order = [c for c in caps if c.endswith("_full_1048576.json")] + \
            [c for c in caps if c.endswith("_full_262144.json")] + \
            [c for c in caps if not c.endswith(("_full_1048576.json", "_full_262144.json"))]
    run = lambda *a: subprocess.run([sys.executable, *a], cwd=ROOT, check=True, capture_output=True)
    run("scripts/ncu_d4_table.py", os.path.join(P, f"{tag}_ncu_d4.md"), *order)
    run("scripts/ncu_source.py", os.path.join(G, "full_1048576.ncu-rep"), os.path.join(P, f"{tag}_source_attr_1M.md"),
        "--envs", "1048576")
    if os.path.exists(os.path.join(G, "fused_1048576.ncu-rep")):
        run("scripts/ncu_source.py", os.path.join(G, "fused_1048576.ncu-rep"),
            os.path.join(P, f"{tag}_fused_source_attr_1M.md"), "--envs", "104857600", "--kernel", "octax_kernel<(int)2")
    wrep = os.path.join(G, "warp_full_pong_standin_4096.ncu-rep")
    if os.path.exists(wrep):
        run("scripts/ncu_source.py", wrep, os.path.join(P, f"{tag}_warp_source_attr_4096.md"), "--envs", "4096",
            "--kernel", "octax_warp_kernel")
    if os.path.exists(os.path.join(G, "launches.csv")):
        run("scripts/ncu_summary.py", "launches", os.path.join(G, "launches.csv"), os.path.join(P, f"{tag}_launches.md"))
    for src, dst in (("paper_protocol.json", "paper_protocol.json"), ("paper_protocol.md", "paper_protocol.md"),
                     ("bench.json", "bench.json"), ("pytest_gpu.log", "pytest_gpu.log"), ("smoke.log", "smoke.log"),
                     ("checked_pytest.log", "checked_build_pytest.log"), ("checked_run.log", "checked_run.log"),
                     ("bench_2rank.json", "bench_2rank_gloo.json")):
        if os.path.exists(os.path.join(G, src)):
            shutil.copy(os.path.join(G, src), os.path.join(P, f"{tag}_{dst}"))
    print(f"{tag}: {len(caps)} captures, digest {have[:16]}")


if __name__ == "__main__":
    main()
