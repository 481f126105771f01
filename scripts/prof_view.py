#!/usr/bin/env python
"""Quick view of an ncu report: key metrics, stall mix, instruction-count groups."""
import csv, collections, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines())); hdr, vals = rows[0], rows[2]
g = lambda m: vals[hdr.index(m)] if m in hdr else "?"
for m in ["gpu__time_duration.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
          "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"]:
    print(f"{m:60s} {g(m)}")
items = [(h, vals[i]) for i, h in enumerate(hdr) if 'smsp__pcsamp_warps_issue_stalled' in h and not h.endswith('not_issued')]
tot = sum(float(v) for h, v in items if v.replace('.', '').isdigit())
print("stalls:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_','')} {float(v)/tot*100:.1f}%"
      for h, v in sorted(items, key=lambda t: -float(t[1]) if t[1].replace('.', '').isdigit() else 0)[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines())); hdr = rows[1]; data = rows[2:]
iex = hdr.index("Instructions Executed"); iss = hdr.index("Warp Stall Sampling (All Samples)")
c = collections.Counter(); s = collections.Counter(); st = collections.Counter()
for r in data:
    e = int(r[iex]); c[e] += 1; s[e] += e; st[e] += int(r[iss])
tot = sum(s.values()); tst = sum(st.values())
for e, k in sorted(s.items(), key=lambda t: -t[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 10]:
    print(f"ex/instr={e:>9}  n_instr={c[e]:>4}  total={k:>11} {k/tot*100:5.1f}%  stall {st[e]/tst*100:5.1f}%")
