#!/usr/bin/env python
"""Per-region attribution of one ncu --set full capture (built with -lineinfo, captured with
--import-source on): executed warp instructions, ALU-pipe instructions (by SASS opcode),
shared-memory excess wavefronts (bank conflicts) and stall samples, summed per source region.

  python scripts/ncu_source.py <prof.ncu-rep> <out.md> [--envs N] [--json out.json]

A region is the span from one marker to the next in the kernel sources: a function
definition (``__device__ ... name(`` / ``__global__``) or a ``// ---- title`` comment, so the
interpreter core's sub-blocks, every DXYN path, the obs copies and the epilogue each get a row.
SASS instructions inlined from another file (octax_dev.cuh) are attributed to that file's
region.  ALU-pipe opcodes follow B300_MICROARCH.md (IADD3/LOP3/SHF/PRMT/ISETP/SEL/... on the
alu pipe); the total is printed next to ncu's own sm__inst_executed_pipe_alu.sum as a check.
"""
from __future__ import annotations

import collections
import csv
import io
import json
import re
import subprocess
import sys

ALU_OPS = {"IADD3", "LOP3", "SHF", "PRMT", "ISETP", "SEL", "LEA", "FLO", "POPC", "BREV", "MOV", "P2R",
           "R2P", "PLOP3", "IMNMX", "VIMNMX", "IABS", "BMSK", "SGXT", "LOP", "IADD", "ICMP", "CSET",
           "CSETP", "VIADD", "IADD32I", "LOP32I", "ISCADD", "BFE", "BFI", "SHL", "SHR", "FSEL", "FSETP"}


def opcode(sass: str) -> str:
    s = sass.strip()
    if s.startswith("@"):
        s = s.split(None, 1)[1] if " " in s else s
    return s.split(None, 1)[0].split(".")[0] if s else ""


EMBEDDED = {}  # file -> {line: text}, the source the capture was taken from (--import-source on)


def markers(path):
    """(line, title) markers of a source file: from the source embedded in the report when it has
    one (so regions match the profiled build even after the file changed), else the file on disk."""
    out = []
    try:
        lines = open(path).read().splitlines()
    except OSError:
        return out
    fn = re.compile(r"^(?:template\s*<[^>]*>\s*)?(?:__device__|__global__|static|cudaError_t)[^;{]*?\b(\w+)\s*\(")
    for i, l in enumerate(lines, 1):
        m = re.search(r"//\s*----\s*(.+)", l)
        if m:
            out.append((i, m.group(1).strip()[:48]))
            continue
        m = fn.match(l.strip())
        if m and "inline" not in m.group(1):
            out.append((i, m.group(1) + "()"))
        elif re.match(r"^\s*(?:__device__\s+)?(?:__noinline__|__forceinline__)", l) or " octax_kernel(" in l \
                or re.match(r"^\s*\w[\w\s<>:*&]*\b(\w+)\(const __grid_constant__", l):
            m2 = re.search(r"\b(\w+)\s*\(", l.split("__forceinline__")[-1].split("__noinline__")[-1])
            if m2:
                out.append((i, m2.group(1) + "()"))
    # the kernel's signature line `octax_kernel(const __grid_constant__ ...`
    for i, l in enumerate(lines, 1):
        if l.startswith("octax_kernel(") or l.startswith("reset_kernel("):
            out.append((i, l.split("(")[0] + "()"))
    return sorted(set(out))


REMAP = {}  # file -> {line in the profiled build: line in the file on disk}


def remap_lines(path):
    """Map the profiled build's line numbers (source embedded in the report: only lines that carry
    code) onto the file on disk by matching line texts near a running offset, so the region
    markers (comments, which the report does not embed) still apply after the file changed."""
    emb = EMBEDDED.get(path)
    try:
        cur = open(path).read().splitlines()
    except OSError:
        return {}
    if not emb:
        return {}
    m, off = {}, 0
    for ln in sorted(emb):
        t = emb[ln].strip()
        j = ln + off - 1
        if 0 <= j < len(cur) and cur[j].strip() == t:
            m[ln] = j + 1
            continue
        best = None
        for d in range(1, 200):
            for k in (j - d, j + d):
                if 0 <= k < len(cur) and t and cur[k].strip() == t:
                    best = k
                    break
            if best is not None:
                break
        if best is not None:
            off = best - (ln - 1)
            m[ln] = best + 1
        else:
            m[ln] = ln + off
    return m


def region_of(file, line, cache):
    if file not in REMAP:
        REMAP[file] = remap_lines(file)
    line = REMAP[file].get(line, line)
    if file not in cache:
        cache[file] = markers(file)
    best = None
    for ln, title in cache[file]:
        if ln <= line:
            best = (ln, title)
        else:
            break
    short = file.rsplit("/", 1)[-1]
    return f"{short}:{best[0]} {best[1]}" if best else f"{short}:? (top)"


def main():
    rep, out = sys.argv[1], sys.argv[2]
    envs = int(sys.argv[sys.argv.index("--envs") + 1]) if "--envs" in sys.argv else None
    jout = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    kfilter = sys.argv[sys.argv.index("--kernel") + 1] if "--kernel" in sys.argv else "octax_kernel"
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    alu_total = None
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) >= 3:
        hdr = rr[0]
        for row in rr[2:]:
            if kfilter in ",".join(row):
                try:  # ALU pipe peak = 2 warp instr / SM / cycle (4 SMSPs x 1 per 2 cycles)
                    pct = float(row[hdr.index("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active")])
                    alu_total = pct / 100.0 * 2.0 * float(row[hdr.index("sm__cycles_active.sum")])
                except (ValueError, IndexError):
                    pass
                break
    efile = None
    for row in csv.reader(io.StringIO(txt)):
        if row and row[0] == "File Path":
            efile = row[1]
        elif row and row[0].isdigit() and len(row) > 1 and efile:
            EMBEDDED.setdefault(efile, {})[int(row[0])] = row[1]
    seen = set()  # an address listed under two source lines (inlining) counts once
    agg = collections.defaultdict(lambda: collections.Counter())
    ops = collections.defaultdict(collections.Counter)
    cache = {}
    file = None
    line = None
    hdr = None
    keep = True
    for row in csv.reader(io.StringIO(txt)):
        if not row:
            continue
        if row[0] == "File Path":
            file = row[1]
            continue
        if row[0] == "Function Name":
            keep = kfilter in row[1]
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or not keep:
            continue
        if row[0] != "":
            try:
                line = int(row[0])
            except ValueError:
                pass
            continue
        if len(row) < len(hdr) or row[3] in ("...", "") or row[2] in seen:
            continue
        seen.add(row[2])
        rec = dict(zip(hdr[2:], row[2:]))
        try:
            ie = float(rec["Instructions Executed"])
        except (KeyError, ValueError):
            continue
        if ie == 0 and rec.get("Warp Stall Sampling (All Samples)", "0") in ("0", "-"):
            continue
        reg = region_of(file, line, cache)
        op = opcode(row[3])
        c = agg[reg]
        c["warp_instr"] += ie
        if op in ALU_OPS:
            c["alu_instr"] += ie
        try:
            c["smem_excess_wavefronts"] += float(rec.get("L1 Wavefronts Shared Excessive", "0") or 0)
            c["stall_samples"] += float(rec.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            pass
        ops[reg][op] += ie
    tot = collections.Counter()
    for c in agg.values():
        tot.update(c)
    rows = sorted(agg.items(), key=lambda kv: -kv[1]["warp_instr"])
    per = (lambda v: v / envs) if envs else (lambda v: v)
    unit = "per env step" if envs else "per launch"
    lines = [f"# ncu source attribution: `{rep}`", "",
             f"Warp instructions and ALU-pipe warp instructions {unit}; shared-memory excess wavefronts "
             "(bank conflicts) and stall samples per launch.  ALU-pipe total by opcode class: "
             f"{per(tot['alu_instr']):.1f} {unit}; ncu's sm__inst_executed_pipe_alu.sum: "
             f"{per(alu_total) if alu_total else float('nan'):.1f}.", "",
             "| region (file:line marker) | warp instr | ALU instr | share of ALU | smem excess wavefronts | stall samples | top opcodes |",
             "|---|---|---|---|---|---|---|"]
    js = []
    for reg, c in rows:
        if c["warp_instr"] < 1e-4 * tot["warp_instr"] and c["smem_excess_wavefronts"] == 0:
            continue
        top = ", ".join(f"{o} {per(v):.1f}" for o, v in ops[reg].most_common(5))
        lines.append(f"| {reg} | {per(c['warp_instr']):.1f} | {per(c['alu_instr']):.1f} | "
                     f"{c['alu_instr'] / max(1, tot['alu_instr']):.3f} | {c['smem_excess_wavefronts']:.0f} | "
                     f"{c['stall_samples']:.0f} | {top} |")
        js.append({"region": reg, "warp_instr": per(c["warp_instr"]), "alu_instr": per(c["alu_instr"]),
                   "smem_excess_wavefronts": c["smem_excess_wavefronts"], "stall_samples": c["stall_samples"],
                   "top_opcodes": {o: per(v) for o, v in ops[reg].most_common(8)}})
    lines.append(f"| **total** | {per(tot['warp_instr']):.1f} | {per(tot['alu_instr']):.1f} | 1 | "
                 f"{tot['smem_excess_wavefronts']:.0f} | {tot['stall_samples']:.0f} | |")
    open(out, "w").write("\n".join(lines) + "\n")
    if jout:
        json.dump({"rep": rep, "envs": envs, "alu_pipe_ncu": alu_total, "regions": js}, open(jout, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
