#!/usr/bin/env python
"""Summarise ncu outputs into profiles/ (committed evidence).

  python scripts/ncu_summary.py launches <launches.csv> <out.md>
  python scripts/ncu_summary.py full <prof.ncu-rep> <out.json> [--envs N] [--game G]
"""
from __future__ import annotations

import collections
import csv
import json
import subprocess
import sys

KEY_METRICS = [
    "gpu__time_duration.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__cycles_active.sum",
    "sm__inst_executed_pipe_fma.sum",
    "smsp__inst_executed.sum",
    "smsp__thread_inst_executed.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_local_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum",
    "l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum",
    "smsp__sass_branch_targets_threads_divergent.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers",
    "launch__grid_size",
    "launch__block_size",
    "sm__cycles_elapsed.avg.per_second",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in data:
        name = r[ik].split("(")[0].replace("void ", "")
        tot[name] += float(r[iv])
        cnt[name] += 1
    allns = sum(tot.values())
    lines = ["| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k, v in tot.most_common():
        lines.append(f"| `{k}` | {cnt[k]} | {v / 1e3:.1f} | {v / cnt[k] / 1e3:.1f} | {v / allns * 100:.1f}% |")
    text = "\n".join(lines)
    with open(out, "w") as f:
        f.write(f"# ncu launch list ({path})\n\n`gpu__time_duration.sum`, cold-cache and serialised "
                "under ncu: compare shares, not absolutes.\n\n" + text + "\n")
    print(text)


def full(path, out, extra):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    res = []
    for v in vals:
        d = {"kernel": v[hdr.index("Kernel Name")][:80]}
        for m in KEY_METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = {"value": v[i], "unit": units[i]}
        res.append(d)
    js = {"source": path, **extra, "launches": res}
    # provenance: the kernel symbol profiled and the device-code digest of the library that ran
    # it (bench.py reports instruction-count rooflines only when both match the loaded build)
    if res:
        js["kernel_symbol"] = res[0]["kernel"]
    so = extra.pop("so", None) if isinstance(extra, dict) else None
    js.pop("so", None)
    if so:
        sys.path.insert(0, ".")
        from paper_2510_01764_b200.build import device_code_digest
        js["sass_sha256"] = device_code_digest(so)
        js["so"] = so
    if res:
        r0 = res[0]
        try:
            rb = float(r0["dram__bytes_read.sum"]["value"]) * (1e6 if r0["dram__bytes_read.sum"]["unit"] == "Mbyte" else 1e9 if r0["dram__bytes_read.sum"]["unit"] == "Gbyte" else 1e3 if r0["dram__bytes_read.sum"]["unit"] == "Kbyte" else 1)
            wb = float(r0["dram__bytes_write.sum"]["value"]) * (1e6 if r0["dram__bytes_write.sum"]["unit"] == "Mbyte" else 1e9 if r0["dram__bytes_write.sum"]["unit"] == "Gbyte" else 1e3 if r0["dram__bytes_write.sum"]["unit"] == "Kbyte" else 1)
            js["dram_bytes_per_launch"] = rb + wb
        except Exception:
            pass
    if res and "envs" in extra:
        try:
            r0 = res[0]
            js["warp_instr_per_env_step"] = float(r0["smsp__inst_executed.sum"]["value"]) / extra["envs"]
            js["warp_exec_efficiency"] = float(r0["smsp__thread_inst_executed_per_inst_executed.ratio"]["value"]) / 32
            pct = float(r0["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"]["value"])
            js["alu_pipe_pct_of_peak"] = pct
            if "sm__inst_executed_pipe_alu.sum" in r0:
                alu = float(r0["sm__inst_executed_pipe_alu.sum"]["value"])
            else:  # ALU pipe peak = 2 warp instr / SM / cycle (4 SMSPs x 1 per 2 cycles)
                alu = pct / 100.0 * 2.0 * float(r0["sm__cycles_active.sum"]["value"])
            js["alu_warp_instr_per_env_step"] = alu / extra["envs"]
            if "dram_bytes_per_launch" in js:
                js["dram_bytes_per_env_step"] = js["dram_bytes_per_launch"] / extra["envs"]
        except Exception:
            pass
    with open(out, "w") as f:
        json.dump(js, f, indent=1)
    for d in res:
        for k, v in d.items():
            print(k, v)


if __name__ == "__main__":
    mode, a, b = sys.argv[1:4]
    extra = {}
    args = sys.argv[4:]
    for k in range(0, len(args) - 1, 2):
        extra[args[k].lstrip("-")] = int(args[k + 1]) if args[k + 1].isdigit() else args[k + 1]
    (launches if mode == "launches" else full)(a, b, *([extra] if mode == "full" else []))
