"""Test helpers: canonical-state construction (SURVEY c.6 layout) and golden
file parsing.  Shared by oracle pins and GPU parity tests; holds no method
arithmetic (only byte layout of the canonical state)."""
from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CANON = 5200


def canon(V=None, I=0, PC=0x200, SP=0, DT=0, ST=0, halted=0, stack=None, draw=0,
          episode=0, steps=0, prev_score=0, ep_ret=0, display=None, hist=None, mem=None):
    c = np.zeros(CANON, np.uint8)
    if V is not None:
        c[0:16] = np.array(V, np.uint8)
    c[16:18] = np.frombuffer(np.uint16(I).tobytes(), np.uint8)
    c[18:20] = np.frombuffer(np.uint16(PC).tobytes(), np.uint8)
    c[20], c[21], c[22], c[23] = SP, DT, ST, halted
    if stack is not None:
        c[24:56] = np.frombuffer(np.array(stack, np.uint16).tobytes(), np.uint8)
    for off, v in ((56, draw), (60, episode), (64, steps), (68, prev_score)):
        c[off:off + 4] = np.frombuffer(np.uint32(v).tobytes(), np.uint8)
    c[72:76] = np.frombuffer(np.int32(ep_ret).tobytes(), np.uint8)
    if display is not None:
        c[80:336] = np.asarray(display, np.uint8).reshape(256)
    if hist is not None:
        c[336:1104] = np.asarray(hist, np.uint8).reshape(768)
    if mem is not None:
        c[1104:5200] = np.asarray(mem, np.uint8)
    return c


def golden_lines(name: str):
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                yield line


def parse_fields(s: str) -> dict:
    out = {}
    for tok in s.split():
        k, v = tok.split("=")
        out[k] = int(v, 0)
    return out


def hand_vectors():
    for line in golden_lines("hand_vectors.txt"):
        op, init, exp = [p.strip() for p in line.split("|")]
        yield int(op, 0), parse_fields(init), parse_fields(exp)


def pristine_mem(rom: bytes, font: bytes) -> np.ndarray:
    m = np.zeros(4096, np.uint8)
    m[0x50:0x50 + len(font)] = np.frombuffer(font, np.uint8)
    m[0x200:0x200 + len(rom)] = np.frombuffer(rom, np.uint8)
    return m
