"""Octo-subset assembler (closed construct list in SURVEY
Appendix E) -- an input generator that turns the paper's Target Shooter
listings into ROM bytes.

The paper names the Octo language but does not define it; the
lowering below follows the CHIP-8 definition and is pinned by behaviour tests
(tests/test_target_shooter.py):

* program layout: ``jump main`` at 0x200, then everything in source order;
* ``: name`` label, ``:alias name vX``, ``:const NAME n``, bare numbers = data bytes;
* ``vX := n | vY | random n | delay``; ``delay := vX``; ``buzzer := vX``;
  ``i := label``; ``vX += n | vY``; ``vX -= vY``;
* ``clear``, ``sprite vX vY n``, ``return`` / ``;``, ``jump label``, bare label = call;
* ``loop ... again`` (nestable); ``if C then S`` where S is one statement
  (including ``again``).  ``if C then S`` executes S iff C: a skip instruction
  tests NOT C.  ``==, !=`` and ``key, -key`` are single skips; ``>=, <=, >`` are
  unsigned compares lowered through VF (VF is clobbered, as in Octo):

      vX >= n   ->  vF := n ; vF =- vX  (8FX7: VF = [vX >= n]) ; skip if VF != 1
      vX <= n   ->  vF := n ; vF -= vX  (8FX5: VF = [n >= vX]) ; skip if VF != 1
      vX >  n   ->  vF := n ; vF -= vX  (VF = [n >= vX])       ; skip if VF != 0
      vX >  vY  ->  vF := vY ; vF -= vX (VF = [vY >= vX])      ; skip if VF != 0

Only encodes instruction words; holds none of the method's arithmetic.
"""
from __future__ import annotations

import re


class OctoError(ValueError):
    pass


_REG = re.compile(r"^v([0-9a-f])$", re.I)


def _tokens(text: str) -> list[str]:
    toks = []
    for line in text.splitlines():
        line = line.split("#", 1)[0]
        toks.extend(line.split())
    return toks


class _Octo:
    def __init__(self, text: str):
        self.toks = _tokens(text)
        self.labels: dict[str, int] = {}
        self.consts: dict[str, int] = {}
        self.aliases: dict[str, int] = {}

    # ---- operand helpers
    def reg(self, t: str) -> int | None:
        if t in self.aliases:
            return self.aliases[t]
        m = _REG.match(t)
        return int(m.group(1), 16) if m else None

    def num(self, t: str, final: bool) -> int:
        if t in self.consts:
            return self.consts[t]
        if t in self.labels:
            return self.labels[t]
        try:
            if t.lower().startswith("0b"):
                return int(t[2:], 2)
            if t.lower().startswith("-0x"):
                return -int(t[3:], 16)
            return int(t, 0)
        except ValueError:
            if final:
                raise OctoError(f"unknown value {t!r}") from None
            return 0

    def is_value(self, t: str) -> bool:
        return (t in self.consts or re.match(r"^-?(0x[0-9a-f]+|0b[01]+|\d+)$", t, re.I) is not None)

    # ---- assembly
    def run(self, final: bool) -> bytearray:
        out = bytearray()
        pc = 0x200 + 2  # 0x200 holds `jump main`
        toks = self.toks
        i = 0
        loops: list[int] = []

        def emit(w: int):
            nonlocal pc
            out.extend([(w >> 8) & 0xFF, w & 0xFF])
            pc += 2

        def need_reg(t):
            r = self.reg(t)
            if r is None:
                raise OctoError(f"expected a register, got {t!r}")
            return r

        def byte(v):
            if final and not -128 <= v <= 255:
                raise OctoError(f"byte out of range: {v}")
            return v & 0xFF

        def addr(t):
            a = self.num(t, final)
            if final and not 0 <= a <= 0xFFF:
                raise OctoError(f"address out of range: {t}")
            return a & 0xFFF

        def statement(j: int) -> int:
            """Emit one statement starting at token j; return the next index."""
            t = toks[j]
            if t in ("return", ";"):
                emit(0x00EE)
                return j + 1
            if t == "clear":
                emit(0x00E0)
                return j + 1
            if t == "jump":
                emit(0x1000 | addr(toks[j + 1]))
                return j + 2
            if t == "again":
                if not loops:
                    raise OctoError("again without loop")
                emit(0x1000 | loops[-1])
                return j + 1
            if t == "sprite":
                x, y = need_reg(toks[j + 1]), need_reg(toks[j + 2])
                n = self.num(toks[j + 3], final)
                emit(0xD000 | x << 8 | y << 4 | (n & 0xF))
                return j + 4
            if t == "delay" and toks[j + 1] == ":=":
                emit(0xF015 | need_reg(toks[j + 2]) << 8)
                return j + 3
            if t == "buzzer" and toks[j + 1] == ":=":
                emit(0xF018 | need_reg(toks[j + 2]) << 8)
                return j + 3
            if t == "i" and toks[j + 1] == ":=":
                emit(0xA000 | addr(toks[j + 2]))
                return j + 3
            x = self.reg(t)
            if x is not None:
                op, rhs = toks[j + 1], toks[j + 2]
                if op == ":=":
                    if rhs == "random":
                        emit(0xC000 | x << 8 | byte(self.num(toks[j + 3], final)))
                        return j + 4
                    if rhs == "delay":
                        emit(0xF007 | x << 8)
                        return j + 3
                    y = self.reg(rhs)
                    if y is not None:
                        emit(0x8000 | x << 8 | y << 4)
                    else:
                        emit(0x6000 | x << 8 | byte(self.num(rhs, final)))
                    return j + 3
                if op == "+=":
                    y = self.reg(rhs)
                    if y is not None:
                        emit(0x8004 | x << 8 | y << 4)
                    else:
                        emit(0x7000 | x << 8 | byte(self.num(rhs, final)))
                    return j + 3
                if op == "-=":
                    emit(0x8005 | x << 8 | need_reg(rhs) << 4)
                    return j + 3
                if op == "=-":
                    emit(0x8007 | x << 8 | need_reg(rhs) << 4)
                    return j + 3
                raise OctoError(f"unsupported register statement {t} {op}")
            if not final or t in self.labels:
                emit(0x2000 | addr(t))  # bare label: subroutine call
                return j + 1
            raise OctoError(f"unknown statement {t!r}")

        while i < len(toks):
            t = toks[i]
            if t == ":":
                name = toks[i + 1]
                if not final:
                    if name in self.labels:
                        raise OctoError(f"duplicate label {name}")
                    self.labels[name] = pc
                i += 2
                continue
            if t == ":alias":
                self.aliases[toks[i + 1]] = need_reg(toks[i + 2])
                i += 3
                continue
            if t == ":const":
                self.consts[toks[i + 1]] = self.num(toks[i + 2], True)
                i += 3
                continue
            if t == "loop":
                loops.append(pc)
                i += 1
                continue
            if t == "again" and loops:
                emit(0x1000 | loops.pop())
                i += 1
                continue
            if t == "if":
                x = need_reg(toks[i + 1])
                rel = toks[i + 2]
                if rel in ("key", "-key"):
                    emit((0xE0A1 if rel == "key" else 0xE09E) | x << 8)
                    j = i + 3
                else:
                    rhs = toks[i + 3]
                    y = self.reg(rhs)
                    j = i + 4
                    if rel == "==":
                        emit((0x9000 | x << 8 | y << 4) if y is not None else (0x4000 | x << 8 | byte(self.num(rhs, final))))
                    elif rel == "!=":
                        emit((0x5000 | x << 8 | y << 4) if y is not None else (0x3000 | x << 8 | byte(self.num(rhs, final))))
                    elif rel in (">=", "<=", ">"):
                        if y is not None and rel != ">":
                            raise OctoError(f"unsupported comparison {rel} with a register")
                        if y is not None:
                            emit(0x8F00 | y << 4)               # vF := vY
                        else:
                            emit(0x6F00 | byte(self.num(rhs, final)))  # vF := n
                        emit((0x8F07 if rel == ">=" else 0x8F05) | x << 4)
                        emit(0x4F01 if rel in (">=", "<=") else 0x4F00)
                    else:
                        raise OctoError(f"unsupported relation {rel!r}")
                if toks[j] != "then":
                    raise OctoError("expected 'then'")
                j += 1
                if toks[j] == "again":  # conditional loop-back: the loop stays open
                    if not loops:
                        raise OctoError("again without loop")
                    emit(0x1000 | loops[-1])
                    # a conditional `again` closes the loop in Octo
                    loops.pop()
                    i = j + 1
                    continue
                i = statement(j)
                continue
            if self.is_value(t) and t not in self.labels:
                out.append(self.num(t, final) & 0xFF)
                pc += 1
                i += 1
                continue
            i = statement(i)
        if loops:
            raise OctoError("unterminated loop")
        return out


def assemble(text: str) -> tuple[bytes, dict[str, int]]:
    """ROM bytes for 0x200 (``jump main`` first) and the label table."""
    a = _Octo(text)
    a.run(final=False)
    a.aliases.clear()
    body = a.run(final=True)
    if "main" not in a.labels:
        raise OctoError("no ': main' label")
    m = a.labels["main"]
    rom = bytes([0x10 | (m >> 8), m & 0xFF]) + bytes(body)
    if len(rom) > 3584:
        raise OctoError("ROM too large")
    return rom, dict(a.labels)
