#!/usr/bin/env python
"""Assemble the paper's Target Shooter L1-L3 listings into roms/*.ch8.

Run on the development box (it reads /root/reference/PAPER.md, which is not
available where tests and the benchmark run):

    python -m workloads.extract_target_shooter [path/to/PAPER.md]

The listings are Appendix D of the paper: level 1 ``lst:level1_code``
(P:536-828), level 2 ``lst:level2_code``, level 3
``lst:level3_code``.  Only the assembled bytes are committed
(with their sha256 in roms/MANIFEST); the listing text stays in the paper.
"""
from __future__ import annotations

import hashlib
import os
import re
import sys

from . import octo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LEVELS = {1: "lst:level1_code", 2: "lst:level2_code", 3: "lst:level3_code"}
CITES = {1: "P:536-828", 2: "P:835-1159", 3: "P:1166-1559"}


def listings(paper: str) -> dict[int, str]:
    text = open(paper).read()
    out = {}
    for lvl, label in LEVELS.items():
        m = re.search(r"\\begin\{lstlisting\}[^\n]*label=\{" + re.escape(label) + r"\}[^\n]*\n(.*?)\\end\{lstlisting\}",
                      text, re.S)
        if not m:
            raise SystemExit(f"listing {label} not found")
        out[lvl] = m.group(1)
    return out


def main(argv):
    paper = argv[1] if len(argv) > 1 else "/root/reference/PAPER.md"
    rom_dir = os.path.join(ROOT, "roms")
    os.makedirs(rom_dir, exist_ok=True)
    lines = []
    for lvl, src in listings(paper).items():
        rom, labels = octo.assemble(src)
        name = f"target_shooter_level{lvl}"
        with open(os.path.join(rom_dir, name + ".ch8"), "wb") as f:
            f.write(rom)
        sha = hashlib.sha256(rom).hexdigest()
        lines.append(f"{name}.ch8 {len(rom)} sha256={sha} source=PAPER.md {CITES[lvl]} "
                     f"(App. D listing {LEVELS[lvl]}), assembled by workloads/octo.py")
        print(name, len(rom), sha[:16], "main at", hex(labels["main"]))
    manifest = os.path.join(rom_dir, "MANIFEST")
    keep = []
    if os.path.exists(manifest):
        keep = [l for l in open(manifest).read().splitlines() if not l.startswith("target_shooter_level")]
    with open(manifest, "w") as f:
        f.write("\n".join(keep + lines) + "\n")


if __name__ == "__main__":
    main(sys.argv)
