"""Workload inputs shared by tests and bench.py: ROM bytes, game specs and
seeded generators.  Plain data and numpy draws only -- none of the method's
arithmetic lives here.

Game specs follow the paper where it gives them (§3.3,
P:1568-1608 App. D) and are labelled "not from paper" otherwise (A8).
"""
from __future__ import annotations

import os

from . import chip8asm, coverage_rom, gen  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
ROM_DIR = os.path.join(os.path.dirname(_HERE), "roms")

# Seeds
ENV_SEED = 0x0C7A_2510_0176_4000
ACTION_SEED = ENV_SEED ^ 0xA5A5_A5A5_A5A5_A5A5

# ---- per-game specs the paper gives -------------------
PAPER_SPECS = {
    # P:152 score V5 ; P:154 terminated V14 == 0 ; keys not in paper
    "brix": {"score": "V5", "terminated": "V14 == 0", "action_keys": None},
    # P:152 score ; P:156 keys {1, 4} ; termination not in paper
    "pong": {"score": "(V14 // 10) - (V14 % 10)", "terminated": "0", "action_keys": [1, 4]},
    # P:154
    "tetris": {"score": None, "terminated": "V1 == 2", "action_keys": None},
    # P:154
    "space_flight": {"score": None, "terminated": "(V9 == 0) | (V12 >= 0x3E)", "action_keys": None},
    # P:156
    "worm": {"score": None, "terminated": None, "action_keys": [2, 4, 6, 8]},
    # P:1577
    "target_shooter": {"score": "V2", "terminated": "V3 == 1", "action_keys": [5, 7, 8, 9, 6]},
}

DEFAULTS = {
    "frame_skip": 4,              # P:228 "each step represents 4 frames"
    "instructions_per_frame": 12,  # A1
    "max_episode_steps": 10000,    # A9
    "quirks": 0,                   # A14 modern profile
    "obs_format": 0,               # packed
    "startup": [],
}


def _src(name: str) -> str:
    with open(os.path.join(_HERE, name)) as f:
        return f.read()


def rom_bytes(name: str) -> bytes:
    """Assemble a stand-in ROM from its committed source (deterministic)."""
    if name == "coverage":
        return coverage_rom.build()[0]
    if name in ("pong_standin", "brix_standin"):
        return chip8asm.assemble(_src(name + ".s"))[0]
    path = os.path.join(ROM_DIR, name + ".ch8")
    with open(path, "rb") as f:
        return f.read()


def game(name: str, **over) -> tuple[bytes, dict]:
    """(ROM, spec) for a named workload."""
    if name == "coverage":
        spec = dict(DEFAULTS, **coverage_rom.SPEC)
    elif name == "pong_standin":
        p = PAPER_SPECS["pong"]
        spec = dict(DEFAULTS, score=p["score"], terminated=p["terminated"],
                    action_keys=p["action_keys"])
    elif name.startswith("target_shooter_level"):
        # the paper's own game (App. D), spec from its wrapper listing:
        # score V[2], terminated V[3] == 1, action_set [5,7,8,9,6]
        p = PAPER_SPECS["target_shooter"]
        spec = dict(DEFAULTS, score=p["score"], terminated=p["terminated"], action_keys=p["action_keys"])
    elif name == "brix_standin":
        p = PAPER_SPECS["brix"]
        spec = dict(DEFAULTS, score=p["score"], terminated=p["terminated"],
                    action_keys=[4, 6])  # not from paper (A8)
    else:
        raise KeyError(name)
    spec.update(over)
    return rom_bytes(name), spec


def n_actions(spec: dict) -> int:
    return len(spec["action_keys"]) + 1
