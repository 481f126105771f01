"""NEXT-1: the Octo-subset assembler and the paper's Target Shooter L1-L3
programs (App. D) as workloads, with behaviour pins taken
from the listings themselves (-m "not gpu")."""
from __future__ import annotations

import hashlib
import os

import numpy as np
import pytest

import oracle
import workloads
from workloads import octo

ROMS = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "roms")
PAPER = "/root/reference/PAPER.md"


def words(rom: bytes):
    return [rom[k] << 8 | rom[k + 1] for k in range(0, len(rom) - 1, 2)]


# ---------------------------------------------------------------- assembler encodings (CHIP-8 definition)
@pytest.mark.parametrize("src,expect", [
    (": main v0 := 5 v1 := v0 v2 += -2 v3 += v1 v4 -= v3 ;",
     [0x1202, 0x6005, 0x8100, 0x72FE, 0x8314, 0x8435, 0x00EE]),
    (": main clear i := main sprite v1 v2 8 delay := v3 buzzer := v4 v5 := delay v6 := random 0x37",
     [0x1202, 0x00E0, 0xA202, 0xD128, 0xF315, 0xF418, 0xF507, 0xC637]),
    # if C then S executes S iff C: the skip tests NOT C
    (": main if v1 == 3 then v2 := 1 if v1 != 3 then v2 := 2 if v1 == v2 then v3 := 0 if v1 != v2 then v3 := 1",
     [0x1202, 0x4103, 0x6201, 0x3103, 0x6202, 0x9120, 0x6300, 0x5120, 0x6301]),
    (": main if v7 key then v0 += 1 if v7 -key then v0 += 2",
     [0x1202, 0xE7A1, 0x7001, 0xE79E, 0x7002]),
    # unsigned compares through VF (module docstring lowering)
    (": main if v7 >= 254 then v7 := 0 if v7 <= 2 then v7 := 3 if v7 > 6 then return if v7 > v8 then return",
     [0x1202, 0x6FFE, 0x8F77, 0x4F01, 0x6700, 0x6F02, 0x8F75, 0x4F01, 0x6703,
      0x6F06, 0x8F75, 0x4F00, 0x00EE, 0x8F80, 0x8F75, 0x4F00, 0x00EE]),
    # loops, conditional again, calls, forward jumps, aliases, consts, data bytes
    (": sub ; : main :alias t v7 :const K 9 loop t := delay if t != 0 then again sub jump end : end 0b10000001 K",
     [0x1204, 0x00EE, 0xF707, 0x3700, 0x1204, 0x2202, 0x120E, 0x8109]),
])
def test_octo_encodings(src, expect):
    rom, _ = octo.assemble(src)
    assert words(rom) == expect


def test_octo_errors():
    with pytest.raises(octo.OctoError):
        octo.assemble("v0 := 1")                    # no main
    with pytest.raises(octo.OctoError):
        octo.assemble(": main loop v0 := 1")        # unterminated loop


def test_octo_comparisons_semantics_bruteforce():
    """Each lowered comparison executes S exactly when the unsigned relation holds,
    checked by running the assembled code on the oracle for all 256 values."""
    for rel, k in ((">=", 200), ("<=", 17), (">", 6)):
        rom, _ = octo.assemble(f": main if v7 {rel} {k} then v0 := 1 : spin jump spin")
        spec = dict(workloads.DEFAULTS, score="0", terminated="0", action_keys=[1])
        e = oracle.OracleEnv(rom, spec, 1, 0)
        base = oracle.canon_fields(e.get_state(0))
        for v in range(256):
            V = [0] * 16
            V[7] = v
            from tests.helpers import canon
            e.set_state(0, canon(V=V, PC=0x200, mem=base["mem"]))
            e.run_cycles(0, 8)
            got = oracle.canon_fields(e.get_state(0))["V"][0]
            want = {">=": v >= k, "<=": v <= k, ">": v > k}[rel]
            assert got == int(want), (rel, k, v)


# ---------------------------------------------------------------- committed ROMs
def test_committed_roms_match_manifest():
    for line in open(os.path.join(ROMS, "MANIFEST")):
        if not line.startswith("target_shooter_level"):
            continue
        name, size, sha = line.split()[:3]
        data = open(os.path.join(ROMS, name), "rb").read()
        assert len(data) == int(size)
        assert hashlib.sha256(data).hexdigest() == sha.split("=")[1]


@pytest.mark.skipif(not os.path.exists(PAPER), reason="paper only on the development box")
def test_roms_reassemble_from_paper(tmp_path):
    from workloads import extract_target_shooter as ex
    for lvl, src in ex.listings(PAPER).items():
        rom, _ = octo.assemble(src)
        assert rom == open(os.path.join(ROMS, f"target_shooter_level{lvl}.ch8"), "rb").read()


# ---------------------------------------------------------------- behaviour pins from the listings
def _no_reset(lvl):
    rom, spec = workloads.game(f"target_shooter_level{lvl}", terminated="0", max_episode_steps=0)
    return rom, spec


@pytest.mark.parametrize("lvl", [1, 2, 3])
def test_crosshair_bounds_invariant(lvl):
    """P:694-697 (L1), P:1023-1026 (L2), P:1408-1411 (L3): boundary checks keep
    crosshair_x = V0 in [0, 56] and crosshair_y = V1 in [0, 24]."""
    rom, spec = workloads.game(f"target_shooter_level{lvl}")
    n = 32
    e = oracle.OracleEnv(rom, spec, n, lvl)
    for t in range(300):
        e.step(workloads.gen.actions(lvl, t, n, 6))
        if t % 10 == 0:
            for j in range(n):
                f = oracle.canon_fields(e.get_state(j))
                assert 0 <= f["V"][0] <= 56 and 0 <= f["V"][1] <= 24


@pytest.mark.parametrize("lvl", [2, 3])
def test_l2_l3_game_over_after_ten_targets(lvl):
    """P:928 / P:1263: the game ends (V3 = 1) once targets_total (VA) reaches 10
    (MAX_TARGETS), hit or missed; the score V2 never exceeds 10."""
    rom, spec = _no_reset(lvl)
    n = 16
    e = oracle.OracleEnv(rom, spec, n, 5)
    ended = np.zeros(n, bool)
    for t in range(2000):
        e.step(workloads.gen.actions(3, t, n, 6))
        for j in range(n):
            f = oracle.canon_fields(e.get_state(j))
            assert f["V"][2] <= 10 and f["V"][10] <= 10
            if f["V"][3] == 1:
                assert f["V"][10] == 10
                ended[j] = True
        if ended.all():
            break
    assert ended.all()


def test_l1_scripted_player_finishes_with_return_ten():
    """P:623/P:646/P:810-811: L1 ends only after targets_hit (VA) == 10 and each hit
    adds exactly 1 to V2, so a terminated L1 episode has return exactly 10.  A
    scripted player (reads the target position from the VM state) drives it."""
    rom, spec = workloads.game("target_shooter_level1", max_episode_steps=0)
    e = oracle.OracleEnv(rom, spec, 1, 99)
    keys = spec["action_keys"]  # [5 up, 7 left, 8 down, 9 right, 6 shoot]
    total, done = 0.0, False
    for t in range(6000):
        f = oracle.canon_fields(e.get_state(0))
        cx, cy, tx, ty, active = f["V"][0], f["V"][1], f["V"][4], f["V"][5], f["V"][6]
        if active and cx + 1 < tx:
            a = keys.index(9) + 1
        elif active and cx > tx + 1:
            a = keys.index(7) + 1
        elif active and cy + 1 < ty:
            a = keys.index(8) + 1
        elif active and cy > ty + 1:
            a = keys.index(5) + 1
        else:
            a = keys.index(6) + 1 if active else 0
        _, r, d, term, _ = e.step(np.array([a], np.int32))
        total += float(r[0])
        if d[0]:
            assert term[0] == 1
            done = True
            break
    assert done and total == 10.0


def test_random_0x37_subset():
    """`target_x := random 0x37` ANDs the random byte with 0x37, so spawned
    targets sit at x in {v : v & ~0x37 == 0}, or 3 after the edge fix-up."""
    rom, spec = _no_reset(1)
    n = 200
    e = oracle.OracleEnv(rom, spec, n, 123)
    for t in range(3):
        e.step(np.zeros(n, np.int32))
    xs = {oracle.canon_fields(e.get_state(j))["V"][4] for j in range(n)}
    assert all((x & ~0x37) == 0 or x == 3 for x in xs)
    assert len(xs) > 10
