#!/usr/bin/env python
"""SURVEY d.4 evidence table from `scripts/ncu_summary.py full` outputs (one column per capture).

    python scripts/ncu_d4_table.py <out.md> <step_full_A.json> [<step_full_B.json> ...]
"""
from __future__ import annotations

import json
import sys

ROWS = [
    ("warp execution efficiency (active lanes / 32)", "smsp__thread_inst_executed_per_inst_executed.ratio", 1 / 32),
    ("issue-slot utilisation, % of peak (active)", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("warp instructions / cycle / SM", "sm__inst_executed.avg.per_cycle_active", 1),
    ("ALU-pipe utilisation, % of peak (active)", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
    ("FMA-pipe utilisation, % of peak (IMAD)", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
    ("LSU-pipe utilisation, % of peak", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
    ("DRAM read", "dram__bytes_read.sum", None),
    ("DRAM write", "dram__bytes_write.sum", None),
    ("DRAM throughput, % of peak (elapsed)", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("shared-memory bank conflicts, loads", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", None),
    ("shared-memory bank conflicts, stores", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", None),
    ("local-memory (spill) requests, loads", "l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum", None),
    ("local-memory (spill) requests, stores", "l1tex__t_requests_pipe_lsu_mem_local_op_st.sum", None),
    ("divergent branch targets", "smsp__sass_branch_targets_threads_divergent.sum", None),
    ("occupancy: active warps, % of 64 / SM", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("registers / thread", "launch__registers_per_thread", None),
    ("kernel time", "gpu__time_duration.sum", None),
]


def main():
    out, files = sys.argv[1], sys.argv[2:]
    caps = [json.load(open(f)) for f in files]
    kind = lambda c: " (warp-per-env)" if "warp_kernel" in str(c.get("kernel_symbol")) else ""  # noqa: E731
    hdr = "| metric (ncu name) | " + " | ".join(f"{c.get('game')} @ {c.get('envs'):,} envs{kind(c)}" for c in caps) + " |"
    lines = [hdr, "|---" * (len(caps) + 1) + "|"]
    for label, m, scale in ROWS:
        cells = []
        for c in caps:
            v = c["launches"][0].get(m)
            if not v:
                cells.append("-")
                continue
            if scale is None:
                cells.append(f"{v['value']} {v['unit']}".strip())
            else:
                cells.append(f"{float(v['value']) * scale:.3f}")
        lines.append(f"| {label} (`{m}`) | " + " | ".join(cells) + " |")
    derived = [("warp instructions / env step", "warp_instr_per_env_step"),
               ("ALU-pipe warp instructions / env step", "alu_warp_instr_per_env_step"),
               ("DRAM bytes / env step (algorithmic: 2,201)", "dram_bytes_per_env_step")]
    for label, k in derived:
        lines.append(f"| {label} | " + " | ".join(f"{c.get(k, float('nan')):.1f}" for c in caps) + " |")
    lines.append("| device-code digest (cuobjdump -sass sha256) | " +
                 " | ".join(str(c.get("sass_sha256"))[:16] for c in caps) + " |")
    with open(out, "w") as f:
        f.write("# SURVEY d.4 ncu evidence (`ncu --set full --clock-control none`, one step launch)\n\n"
                + "\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
