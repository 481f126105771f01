"""Tiny two-pass CHIP-8 assembler (host tool for authoring test ROMs).

This is an input generator: it turns mnemonic text into ROM bytes that both
the oracle and the CUDA path then execute.  It contains no part of the
method's arithmetic (it only *encodes* instruction words; decoding and
execution live separately in oracle/ and paper_2510_01764_b200/csrc/).

Syntax (Cowgod-style mnemonics, one statement per line)::

    ; comment            # comment
    label:               .equ NAME expr        .org addr
    .db e, e, ...        .dw e, ...            .fill count, byte
    CLS  RET  SYS a  JP a  JP V0, a  CALL a
    SE Vx, b|Vy   SNE Vx, b|Vy   LD Vx, b|Vy|DT|K|[I]   LD I, a
    LD DT, Vx  LD ST, Vx  LD F, Vx  LD B, Vx  LD [I], Vx
    ADD Vx, b|Vy  ADD I, Vx  OR/AND/XOR/SUB/SUBN Vx, Vy  SHR Vx[, Vy]  SHL Vx[, Vy]
    RND Vx, b  DRW Vx, Vy, n  SKP Vx  SKNP Vx

Expressions: decimal, 0x.., 0b.., labels, .equ names, with + - * and
parentheses-free left-to-right evaluation.
"""
from __future__ import annotations

import re

ROM_BASE = 0x200


class AsmError(ValueError):
    pass


_REG = re.compile(r"^v([0-9a-f])$", re.I)


def _reg(tok: str) -> int | None:
    m = _REG.match(tok.strip())
    return int(m.group(1), 16) if m else None


def _split_operands(s: str) -> list[str]:
    return [t.strip() for t in s.split(",")] if s.strip() else []


class _Asm:
    def __init__(self, text: str):
        self.lines = text.splitlines()
        self.symbols: dict[str, int] = {}

    def value(self, expr: str, final: bool) -> int:
        toks = re.findall(r"0x[0-9a-fA-F]+|0b[01]+|\d+|[A-Za-z_][\w.]*|[+\-*]", expr.replace(" ", ""))
        if not toks:
            raise AsmError(f"empty expression: {expr!r}")
        total, op = 0, "+"
        for t in toks:
            if t in "+-*":
                op = t
                continue
            if t.lower().startswith("0x"):
                v = int(t, 16)
            elif t.lower().startswith("0b"):
                v = int(t[2:], 2)
            elif t.isdigit():
                v = int(t)
            elif t in self.symbols:
                v = self.symbols[t]
            elif not final:
                v = 0
            else:
                raise AsmError(f"undefined symbol {t!r}")
            total = total + v if op == "+" else total - v if op == "-" else total * v
        return total

    def encode(self, mnem: str, ops: list[str], final: bool) -> list[int]:
        m = mnem.upper()
        V = lambda i: _reg(ops[i])
        val = lambda i: self.value(ops[i], final)

        def need(cond: bool):
            if not cond:
                raise AsmError(f"bad operands for {mnem}: {ops}")

        def nnn(i):
            a = val(i)
            if final and not 0 <= a <= 0xFFF:
                raise AsmError(f"address out of range: {ops[i]}")
            return a & 0xFFF

        def byte(i):
            b = val(i)
            if final and not -128 <= b <= 255:
                raise AsmError(f"byte out of range: {ops[i]}")
            return b & 0xFF

        if m == "CLS":
            return [0x00E0]
        if m == "RET":
            return [0x00EE]
        if m == "SYS":
            return [nnn(0)]
        if m == "JP":
            if len(ops) == 2:
                need(V(0) == 0)
                return [0xB000 | nnn(1)]
            return [0x1000 | nnn(0)]
        if m == "CALL":
            return [0x2000 | nnn(0)]
        if m in ("SE", "SNE"):
            x = V(0)
            need(x is not None and len(ops) == 2)
            y = V(1)
            if y is not None:
                return [(0x5000 if m == "SE" else 0x9000) | x << 8 | y << 4]
            return [(0x3000 if m == "SE" else 0x4000) | x << 8 | byte(1)]
        if m == "LD":
            need(len(ops) == 2)
            a, b = ops[0].upper(), ops[1].upper()
            x = V(0)
            if x is not None:
                y = V(1)
                if y is not None:
                    return [0x8000 | x << 8 | y << 4]
                if b == "DT":
                    return [0xF007 | x << 8]
                if b == "K":
                    return [0xF00A | x << 8]
                if b == "[I]":
                    return [0xF065 | x << 8]
                return [0x6000 | x << 8 | byte(1)]
            if a == "I":
                return [0xA000 | nnn(1)]
            y = V(1)
            need(y is not None)
            table = {"DT": 0xF015, "ST": 0xF018, "F": 0xF029, "B": 0xF033, "[I]": 0xF055}
            need(a in table)
            return [table[a] | y << 8]
        if m == "ADD":
            need(len(ops) == 2)
            if ops[0].upper() == "I":
                return [0xF01E | V(1) << 8]
            x = V(0)
            need(x is not None)
            y = V(1)
            if y is not None:
                return [0x8004 | x << 8 | y << 4]
            return [0x7000 | x << 8 | byte(1)]
        alu = {"OR": 1, "AND": 2, "XOR": 3, "SUB": 5, "SHR": 6, "SUBN": 7, "SHL": 0xE}
        if m in alu:
            x = V(0)
            y = V(1) if len(ops) > 1 else 0
            need(x is not None and y is not None)
            return [0x8000 | x << 8 | y << 4 | alu[m]]
        if m == "RND":
            return [0xC000 | V(0) << 8 | byte(1)]
        if m == "DRW":
            n = val(2)
            need(0 <= n <= 15 or not final)
            return [0xD000 | V(0) << 8 | V(1) << 4 | (n & 0xF)]
        if m == "SKP":
            return [0xE09E | V(0) << 8]
        if m == "SKNP":
            return [0xE0A1 | V(0) << 8]
        raise AsmError(f"unknown mnemonic {mnem!r}")

    def run(self, final: bool) -> bytearray:
        out = bytearray()
        pc = ROM_BASE
        for ln, raw in enumerate(self.lines, 1):
            line = re.split(r"[;#]", raw, maxsplit=1)[0].strip()
            try:
                while True:
                    m = re.match(r"^([A-Za-z_][\w.]*):\s*(.*)$", line)
                    if not m:
                        break
                    if not final:
                        if m.group(1) in self.symbols and self.symbols[m.group(1)] != pc:
                            raise AsmError(f"duplicate label {m.group(1)}")
                        self.symbols[m.group(1)] = pc
                    line = m.group(2).strip()
                if not line:
                    continue
                parts = line.split(None, 1)
                mnem, rest = parts[0], (parts[1] if len(parts) > 1 else "")
                ops = _split_operands(rest)
                d = mnem.lower()
                if d == ".equ":
                    name, expr = rest.split(None, 1) if "," not in rest else [t.strip() for t in rest.split(",", 1)]
                    self.symbols[name] = self.value(expr, final)
                    continue
                if d == ".org":
                    target = self.value(ops[0], final)
                    if target < pc:
                        raise AsmError(".org moves backwards")
                    out.extend(b"\x00" * (target - pc))
                    pc = target
                    continue
                if d == ".db":
                    for o in ops:
                        out.append(self.value(o, final) & 0xFF)
                        pc += 1
                    continue
                if d == ".dw":
                    for o in ops:
                        w = self.value(o, final) & 0xFFFF
                        out.extend([w >> 8, w & 0xFF])
                        pc += 2
                    continue
                if d == ".fill":
                    cnt, b = self.value(ops[0], final), self.value(ops[1], final) & 0xFF
                    out.extend([b] * cnt)
                    pc += cnt
                    continue
                for w in self.encode(mnem, ops, final):
                    out.extend([w >> 8, w & 0xFF])
                    pc += 2
            except AsmError as e:
                raise AsmError(f"line {ln}: {e}: {raw.strip()}") from None
            except (TypeError, IndexError):
                raise AsmError(f"line {ln}: bad statement: {raw.strip()}") from None
        return out


def assemble(text: str) -> tuple[bytes, dict[str, int]]:
    """Return (ROM bytes loaded at 0x200, symbol table)."""
    a = _Asm(text)
    a.run(final=False)
    rom = a.run(final=True)
    if not 0 < len(rom) <= 3584:
        raise AsmError(f"ROM size {len(rom)} outside 1..3584")
    return bytes(rom), dict(a.symbols)
