"""ROM tooling: disassembler and the static analyses of the
paper's Appendix B.1 ("scan for FX33 (BCD) to locate score registers")
plus a key-operand scan that derives a game's action set from its EX9E / EXA1
instructions.  Host-side only; results are suggestions labelled "derived, not
from paper" (reading A8), never used by the hot path.

    python -m paper_2510_01764_b200.romtools game.ch8
"""
from __future__ import annotations

import sys
from dataclasses import dataclass, field

BASE = 0x200


def mnemonic(op: int) -> str:
    """Cowgod-style text for one 16-bit word (unknown words -> DW)."""
    hi, x, y, n, nn, nnn = op >> 12, (op >> 8) & 15, (op >> 4) & 15, op & 15, op & 255, op & 0xFFF
    if op == 0x00E0:
        return "CLS"
    if op == 0x00EE:
        return "RET"
    table = {
        0x0: lambda: f"SYS {nnn:#05x}",
        0x1: lambda: f"JP {nnn:#05x}",
        0x2: lambda: f"CALL {nnn:#05x}",
        0x3: lambda: f"SE V{x:X}, {nn:#04x}",
        0x4: lambda: f"SNE V{x:X}, {nn:#04x}",
        0x6: lambda: f"LD V{x:X}, {nn:#04x}",
        0x7: lambda: f"ADD V{x:X}, {nn:#04x}",
        0xA: lambda: f"LD I, {nnn:#05x}",
        0xB: lambda: f"JP V0, {nnn:#05x}",
        0xC: lambda: f"RND V{x:X}, {nn:#04x}",
        0xD: lambda: f"DRW V{x:X}, V{y:X}, {n}",
    }
    if hi in table:
        return table[hi]()
    if hi == 0x5 and n == 0:
        return f"SE V{x:X}, V{y:X}"
    if hi == 0x9 and n == 0:
        return f"SNE V{x:X}, V{y:X}"
    if hi == 0x8:
        alu = {0: "LD", 1: "OR", 2: "AND", 3: "XOR", 4: "ADD", 5: "SUB", 6: "SHR", 7: "SUBN", 0xE: "SHL"}
        if n in alu:
            return f"{alu[n]} V{x:X}, V{y:X}"
    if hi == 0xE and nn in (0x9E, 0xA1):
        return f"{'SKP' if nn == 0x9E else 'SKNP'} V{x:X}"
    if hi == 0xF:
        f = {0x07: f"LD V{x:X}, DT", 0x0A: f"LD V{x:X}, K", 0x15: f"LD DT, V{x:X}", 0x18: f"LD ST, V{x:X}",
             0x1E: f"ADD I, V{x:X}", 0x29: f"LD F, V{x:X}", 0x33: f"LD B, V{x:X}", 0x55: f"LD [I], V{x:X}",
             0x65: f"LD V{x:X}, [I]"}
        if nn in f:
            return f[nn]
    return f"DW {op:#06x}"


def _word(rom: bytes, addr: int) -> int | None:
    k = addr - BASE
    if k < 0 or k + 1 >= len(rom):
        return None
    return rom[k] << 8 | rom[k + 1]


def reachable(rom: bytes) -> list[int]:
    """Code addresses reachable from 0x200 by following fall-through, skips, jumps
    and calls (recursive traversal).  BNNN is treated as a jump table: the first
    8 words at NNN are followed (a heuristic; V0 is not known statically)."""
    seen, todo = set(), [BASE]
    while todo:
        a = todo.pop()
        while a not in seen:
            w = _word(rom, a)
            if w is None:
                break
            seen.add(a)
            hi = w >> 12
            if hi == 0x1:
                todo.append(w & 0xFFF)
                break
            if hi == 0x2:
                todo.append(w & 0xFFF)
            if hi == 0xB:
                todo.extend((w & 0xFFF) + 2 * k for k in range(8))
                break
            if w == 0x00EE:
                break
            if hi in (0x3, 0x4, 0x5, 0x9) or (hi == 0xE and (w & 0xFF) in (0x9E, 0xA1)):
                todo.append(a + 4)  # skip target
            a += 2
    return sorted(seen)


def disassemble(rom: bytes, linear: bool = False) -> list[tuple[int, int, str]]:
    addrs = range(BASE, BASE + len(rom) - 1, 2) if linear else reachable(rom)
    return [(a, _word(rom, a), mnemonic(_word(rom, a))) for a in addrs]


@dataclass
class RomFacts:
    bcd_registers: list = field(default_factory=list)   # FX33 operands (score candidates)
    key_registers: list = field(default_factory=list)   # EX9E / EXA1 operands
    keys: list = field(default_factory=list)            # immediates loaded into those registers
    waits_for_key: bool = False                         # FX0A present
    uses_random: bool = False
    draws: int = 0


def analyse(rom: bytes) -> RomFacts:
    code = disassemble(rom)
    f = RomFacts()
    last_imm: dict[int, int] = {}
    keys = []
    for a, w, _ in code:
        hi, x, nn = w >> 12, (w >> 8) & 15, w & 255
        if hi == 0x6:
            last_imm[x] = nn & 15
        if hi == 0xF and nn == 0x33 and x not in f.bcd_registers:
            f.bcd_registers.append(x)
        if hi == 0xE and nn in (0x9E, 0xA1):
            if x not in f.key_registers:
                f.key_registers.append(x)
            if x in last_imm and last_imm[x] not in keys:
                keys.append(last_imm[x])
        if hi == 0xF and nn == 0x0A:
            f.waits_for_key = True
        if hi == 0xC:
            f.uses_random = True
        if hi == 0xD:
            f.draws += 1
    f.keys = keys
    return f


def suggest_spec(rom: bytes) -> dict:
    """A starting game spec derived from the ROM (labelled: not from paper, A8)."""
    f = analyse(rom)
    spec = {"action_keys": f.keys or list(range(16)), "terminated": "0",
            "score": f"V{f.bcd_registers[0]:X}" if f.bcd_registers else "0",
            "provenance": "derived by romtools.suggest_spec (static scan), not from paper"}
    return spec


def main(argv):
    rom = open(argv[1], "rb").read()
    for a, w, m in disassemble(rom):
        print(f"{a:03X}: {w:04X}  {m}")
    print(analyse(rom))
    print(suggest_spec(rom))


if __name__ == "__main__":
    main(sys.argv)
