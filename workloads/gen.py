"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and
bench.py.  Holds none of the method's arithmetic: only numpy random draws
that produce ROM bytes and action arrays, which are then handed unchanged to
both implementations.

Recipe:
  * actions: uniform over {0..n_actions-1} per env per step (P:226 uses a
    constant action; we add uniform random actions so key handling and
    resets are exercised), from numpy PCG64 seeded per (seed, step).
  * fuzz ROMs: instruction words drawn from a weighted mix of the 35 opcode
    forms (SURVEY c.5), with jump/call targets and I addresses kept inside
    the program/data area so programs run for a long time, a configurable
    rate of self-modifying stores, draws, key polls, CXNN and faults.
"""
from __future__ import annotations

import numpy as np


def actions(seed: int, step: int, n_envs: int, n_actions: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64([seed & 0xFFFFFFFF, step, 0xAC7]))
    return rng.integers(0, n_actions, size=n_envs, dtype=np.int64).astype(np.int32)


def action_stream(seed: int, steps: int, n_envs: int, n_actions: int) -> np.ndarray:
    return np.stack([actions(seed, t, n_envs, n_actions) for t in range(steps)])


def fuzz_rom(seed: int, n_instr: int = 256, fault_rate: float = 0.002,
             smc_rate: float = 0.02, data_bytes: int = 64) -> bytes:
    """A random but long-running CHIP-8 program.

    Layout: 0x200: code (n_instr words), then `data_bytes` of random sprite /
    table data.  Targets of 1NNN/2NNN/BNNN land on code words (even
    offsets, sometimes odd), ANNN points into data, code or font.
    """
    rng = np.random.Generator(np.random.PCG64([seed & 0xFFFFFFFF, 0xF022]))
    code_lo, code_hi = 0x200, 0x200 + 2 * n_instr
    data_lo = code_hi
    r = lambda n: int(rng.integers(0, n))

    def target():
        t = code_lo + 2 * r(n_instr)
        if rng.random() < 0.01:
            t += 1  # odd PC
        return t & 0xFFF

    forms = [
        # (weight, generator)
        (3, lambda: 0x00E0),
        (3, lambda: 0x00EE),
        (1, lambda: r(0x1000) if r(8) else 0x0000),          # 0NNN no-op
        (6, lambda: 0x1000 | target()),
        (4, lambda: 0x2000 | target()),
        (6, lambda: 0x3000 | r(16) << 8 | (r(4) if r(2) else r(256))),
        (6, lambda: 0x4000 | r(16) << 8 | (r(4) if r(2) else r(256))),
        (3, lambda: 0x5000 | r(16) << 8 | r(16) << 4),
        (8, lambda: 0x6000 | r(16) << 8 | r(256)),
        (8, lambda: 0x7000 | r(16) << 8 | r(256)),
        (14, lambda: 0x8000 | r(16) << 8 | r(16) << 4 | [0, 1, 2, 3, 4, 5, 6, 7, 0xE][r(9)]),
        (3, lambda: 0x9000 | r(16) << 8 | r(16) << 4),
        (6, lambda: 0xA000 | (data_lo + r(data_bytes) if r(3) else
                              (0x50 + r(80) if r(2) else code_lo + r(2 * n_instr)))),
        (2, lambda: 0xB000 | ((target() - r(8)) & 0xFFF)),
        (5, lambda: 0xC000 | r(16) << 8 | r(256)),
        (8, lambda: 0xD000 | r(16) << 8 | r(16) << 4 | r(16)),
        (3, lambda: 0xE09E | r(16) << 8),
        (3, lambda: 0xE0A1 | r(16) << 8),
        (2, lambda: 0xF007 | r(16) << 8),
        (1, lambda: 0xF00A | r(16) << 8),
        (2, lambda: 0xF015 | r(16) << 8),
        (1, lambda: 0xF018 | r(16) << 8),
        (2, lambda: 0xF01E | r(16) << 8),
        (2, lambda: 0xF029 | r(16) << 8),
        (2, lambda: 0xF033 | r(16) << 8),
        (2, lambda: 0xF055 | r(16) << 8),
        (2, lambda: 0xF065 | r(16) << 8),
    ]
    w = np.array([f[0] for f in forms], float)
    w /= w.sum()
    words = []
    for _ in range(n_instr):
        u = rng.random()
        if u < fault_rate:
            words.append([0x5001, 0x8008, 0xE000, 0xF0FF, 0x900F][r(5)] | r(16) << 8)
            continue
        if u < fault_rate + smc_rate:
            # point I at code so a following FX55/FX33 rewrites instructions
            words.append(0xA000 | (code_lo + r(2 * n_instr)))
            continue
        words.append(int(forms[int(rng.choice(len(forms), p=w))][1]()))
    rom = bytearray()
    for wd in words:
        rom += bytes([wd >> 8 & 0xFF, wd & 0xFF])
    rom += bytes(int(x) for x in rng.integers(0, 256, size=data_bytes))
    return bytes(rom)
