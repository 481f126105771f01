"""Pins for the CPU oracle (-m "not gpu").

Each test checks the oracle against something other than itself: values the
paper / SPEC / CHIP-8 definition fix (golden files with citations), closed
mathematical counts, invariants, and brute force on tiny inputs.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workloads
from tests.helpers import canon, golden_lines, hand_vectors

SELF_JUMP = bytes([0x12, 0x00])  # 1200: jump to self
BASE_SPEC = dict(workloads.DEFAULTS, score="0", terminated="0", action_keys=[1, 4])


def _env(rom=SELF_JUMP, n=1, seed=42, offset=0, **over):
    return oracle.OracleEnv(rom, dict(BASE_SPEC, **over), n, seed, offset)


def _run_word(env, word, init, keys=0, j=0):
    c = env.get_state(j)
    f = oracle.canon_fields(c)
    mem = f["mem"]
    mem[0x300] = word >> 8
    mem[0x301] = word & 0xFF
    V = list(f["V"])
    for k in range(16):
        if f"V{k:X}" in init:
            V[k] = init[f"V{k:X}"]
        if f"V{k}" in init:
            V[k] = init[f"V{k}"]
    stack = [0] * 16
    if "STK0" in init:
        stack[0] = init["STK0"]
    st = canon(V=V, I=init.get("I", 0), PC=0x300, SP=init.get("SP", 0), DT=init.get("DT", 0),
               ST=init.get("ST", 0), stack=stack, mem=mem)
    env.set_state(j, st)
    env.run_cycles(j, 1, keys)
    return oracle.canon_fields(env.get_state(j))


# ---------------------------------------------------------------- Philox
def test_philox_kat():
    n = 0
    for line in golden_lines("philox_kat.txt"):
        v = [int(t, 16) for t in line.split()]
        assert oracle.philox4x32_10(v[0:4], v[4:6]) == v[6:10]
        n += 1
    assert n == 3


def test_cxnn_uses_philox_mapping():
    """A12: CXNN byte = Philox(ctr={draw, episode, gid, 0}, key=seed).out0 & 0xFF."""
    seed = 0x1234_5678_9ABC_DEF0
    for gid in (0, 7, 123456):
        e = oracle.OracleEnv(bytes([0xC1, 0xFF, 0xC2, 0xFF, 0x12, 0x04]),
                             dict(BASE_SPEC), 1, seed, gid)
        e.run_cycles(0, 2)
        f = oracle.canon_fields(e.get_state(0))
        key = [seed & 0xFFFFFFFF, seed >> 32]
        assert f["V"][1] == oracle.philox4x32_10([0, 0, gid, 0], key)[0] & 0xFF
        assert f["V"][2] == oracle.philox4x32_10([1, 0, gid, 0], key)[0] & 0xFF
        assert f["draw"] == 2


def _mapping(kind):
    for line in golden_lines("philox_mapping.txt"):
        tok = line.split()
        if tok[0] == kind:
            yield tok[1:]


def test_cxnn_mapping_golden_incl_episode_and_gid():
    """SURVEY App. C mapping vectors (tests/golden/philox_mapping.txt): CXNN run by the
    oracle from a set state with the given draw / episode counters and global id (env
    offset) stores exactly the golden byte, so a counter slot swap (draw <-> episode,
    gid in the wrong word) or a wrong domain fails here."""
    rows = list(_mapping("cxnn"))
    assert len(rows) == 5
    for seed, draw, ep, gid, dom, out0, byte in rows:
        seed, draw, ep, gid, dom = (int(v) for v in (seed, draw, ep, gid, dom))
        assert oracle.philox4x32_10([draw, ep, gid, dom], [seed & 0xFFFFFFFF, seed >> 32])[0] == int(out0, 16)
        if dom != 0:
            continue
        e = oracle.OracleEnv(SELF_JUMP, dict(BASE_SPEC), 1, seed, gid)
        f = oracle.canon_fields(e.get_state(0))
        mem = f["mem"]
        mem[0x300], mem[0x301] = 0xC7, 0xFF                 # C7FF: V7 = byte & 0xFF
        e.set_state(0, canon(PC=0x300, draw=draw, episode=ep, mem=mem))
        e.run_cycles(0, 1)
        g = oracle.canon_fields(e.get_state(0))
        assert g["V"][7] == int(byte, 16), (draw, ep, gid)
        assert g["draw"] == draw + 1 and g["episode"] == ep


def test_cxnn_episode_counter_after_auto_reset():
    """The episode slot advances on auto-reset (c.1 step: episode += 1; reset draws restart
    at 0): a startup frame that runs CXNN gives the golden byte of episode 0 at create and of
    episode 1 after the first (always-terminating) step, seed 42, gid 0 (App. C)."""
    want = {int(r[2]): int(r[6], 16) for r in _mapping("cxnn")
            if r[0] == "42" and r[1] == "0" and r[3] == "0" and r[4] == "0"}
    rom = bytes([0xC1, 0xFF, 0x12, 0x02])                 # C1FF ; 1202 (self-jump)
    e = oracle.OracleEnv(rom, dict(BASE_SPEC, terminated="1", startup=[(0, 1)]), 1, 42, 0)
    f = oracle.canon_fields(e.get_state(0))
    assert (f["V"][1], f["episode"], f["draw"]) == (want[0], 0, 1)
    _, _, done, term, _ = e.step(np.zeros(1, np.int32))
    assert done[0] == 1 and term[0] == 1
    f = oracle.canon_fields(e.get_state(0))
    assert (f["V"][1], f["episode"], f["draw"]) == (want[1], 1, 1)


def test_action_stream_golden_table():
    """SURVEY App. C synthetic action table (aseed 42, gids 0-2, t 0-3): out0 and its
    residues mod 3 (Pong) and mod 17 (coverage ROM)."""
    rows = list(_mapping("action"))
    assert len(rows) == 12
    for aseed, gid, t, out0, m3, m17 in rows:
        aseed, gid, t = int(aseed), int(gid), int(t)
        assert oracle.philox4x32_10([t, 0, gid, 1], [aseed, 0])[0] == int(out0, 16)
        assert oracle.synthetic_action(aseed, t, gid, 3) == int(m3)
        assert oracle.synthetic_action(aseed, t, gid, 17) == int(m17)
        assert oracle.synthetic_actions(aseed, t, [gid], 17)[0] == int(m17)


def test_sampled_env_ids_golden():
    """SURVEY App. C config-4 sampled ids (seed 42, n_total 262,144, domain 2, k = 0..4),
    the recipe tests/test_gpu_parity.py uses to pick its sampled envs."""
    rows = list(_mapping("sample"))
    assert len(rows) == 5
    for seed, ntot, k, gid in rows:
        seed = int(seed)
        out0 = oracle.philox4x32_10([int(k), 0, 0, 2], [seed & 0xFFFFFFFF, seed >> 32])[0]
        assert out0 % int(ntot) == int(gid)


def test_synthetic_action_definition():
    for t, gid in ((0, 0), (5, 3), (2**33 + 1, 99)):
        out0 = oracle.philox4x32_10([t & 0xFFFFFFFF, t >> 32, gid, 1], [42, 0])[0]
        assert oracle.synthetic_action(42, t, gid, 17) == out0 % 17


# ---------------------------------------------------------------- load / font / fetch
def test_power_on_layout():
    rom = bytes([0xA2, 0xF0])
    e = _env(rom)
    f = oracle.canon_fields(e.get_state(0))
    assert f["PC"] == 0x200
    assert f["mem"][0x50] == 0xF0                 # S:66 first font byte
    assert f["mem"][0x200] == 0xA2 and f["mem"][0x201] == 0xF0
    font = f["mem"][0x50:0xA0]
    # each glyph is 4 pixels wide: the low nibble of every row is 0 (App. A.4 "4x5")
    assert np.all(font & 0x0F == 0)
    glyphs = {bytes(font[5 * k:5 * k + 5]) for k in range(16)}
    assert len(glyphs) == 16
    assert np.all(f["mem"][:0x50] == 0) and np.all(f["mem"][0xA0:0x200] == 0)
    # fetch A2F0 -> I = 0x2F0, PC = 0x202
    e.run_cycles(0, 1)
    f = oracle.canon_fields(e.get_state(0))
    assert (f["I"], f["PC"]) == (0x2F0, 0x202)


def test_rom_size_bounds():
    rom = bytes([0x12, 0x00]) + bytes(range(256)) * 14
    rom = rom[:3584]
    e = _env(rom)
    assert oracle.canon_fields(e.get_state(0))["mem"][0xFFF] == rom[-1]
    with pytest.raises(oracle.OracleError) as ei:
        _env(rom + b"\x00")
    assert ei.value.code == -3
    with pytest.raises(oracle.OracleError) as ei:
        _env(b"")
    assert ei.value.code == -2


def test_pc_out_of_range_halts():
    e = _env()
    c = e.get_state(0)
    f = oracle.canon_fields(c)
    mem = f["mem"]
    mem[0xFFE], mem[0xFFF] = 0x60, 0x07  # 6007 at 0xFFE is a legal fetch
    e.set_state(0, canon(PC=0xFFE, mem=mem))
    e.run_cycles(0, 1)
    f = oracle.canon_fields(e.get_state(0))
    assert f["V"][0] == 7 and f["PC"] == 0x1000 and not f["halted"]
    e.run_cycles(0, 1)
    assert oracle.canon_fields(e.get_state(0))["halted"] == 1


# ---------------------------------------------------------------- hand vectors
@pytest.mark.parametrize("word,init,exp", list(hand_vectors()))
def test_hand_vector(word, init, exp):
    e = _env()
    f = _run_word(e, word, init, keys=init.get("KEYS", 0))
    for k, v in exp.items():
        if k.startswith("MEM["):
            assert f["mem"][int(k[4:-1], 0)] == v, k
        elif k == "HALT":
            assert f["halted"] == v
        elif k == "STK0":
            assert f["stack"][0] == v
        elif k == "DRAW":
            assert f["draw"] == v
        elif k in ("I", "PC", "SP", "DT", "ST"):
            assert f[k] == v, k
        else:
            assert f["V"][int(k[1:], 16) if not k[1:].isdigit() else int(k[1:])] == v, k


# ---------------------------------------------------------------- exhaustive ALU
def _alu_table(op_n):
    """Run 8 1 2 n for all 65536 (V1, V2) pairs; returns (V1', VF') arrays."""
    e = _env(n=256)
    base = oracle.canon_fields(e.get_state(0))["mem"]
    base[0x300], base[0x301] = 0x81, 0x20 | op_n
    r = np.zeros((256, 256), np.int64)
    vf = np.zeros((256, 256), np.int64)
    for a in range(256):
        for b in range(256):
            V = [0] * 16
            V[1], V[2] = a, b
            e.set_state(b, canon(V=V, PC=0x300, mem=base))
        for b in range(256):
            e.run_cycles(b, 1)
            c = e.get_state(b)
            r[a, b], vf[a, b] = c[1], c[15]
    return r, vf


@pytest.mark.slow
def test_exhaustive_alu_counts_and_inverses():
    A, B = np.meshgrid(np.arange(256), np.arange(256), indexing="ij")
    r4, f4 = _alu_table(4)
    assert f4.sum() == 32640                     # #{(a,b): a+b >= 256} = 255*256/2
    assert np.all(r4 + 256 * f4 == A + B)         # exact 9-bit sum decomposition
    r5, f5 = _alu_table(5)
    assert f5.sum() == 32896                     # #{(a,b): a >= b} = 256*257/2
    assert np.all((r5 + B) % 256 == A)            # inverse of subtraction
    assert np.all(f5[A >= B] == 1) and np.all(f5[A < B] == 0)
    r7, f7 = _alu_table(7)
    assert f7.sum() == 32896
    assert np.all((r7 + A) % 256 == B)
    r6, f6 = _alu_table(6)
    assert np.all(2 * r6 + f6 == A)               # shifted-out bit reconstructs VX
    rE, fE = _alu_table(0xE)
    assert np.all((rE >> 1) + 128 * fE == A)
    assert fE.sum() == 128 * 256 and f6.sum() == 128 * 256


# ---------------------------------------------------------------- decode totality
def _valid_word(w: int) -> bool:
    """The 35-instruction ISA table (SURVEY c.5 / S:158), as an enumeration."""
    hi, x, nn, n = w >> 12, (w >> 8) & 0xF, w & 0xFF, w & 0xF
    if hi in (0x0, 0x1, 0x2, 0x3, 0x4, 0x6, 0x7, 0xA, 0xB, 0xC, 0xD):
        return True
    if hi in (0x5, 0x9):
        return n == 0
    if hi == 0x8:
        return n in (0, 1, 2, 3, 4, 5, 6, 7, 0xE)
    if hi == 0xE:
        return nn in (0x9E, 0xA1)
    return nn in (0x07, 0x0A, 0x15, 0x18, 0x1E, 0x29, 0x33, 0x55, 0x65)


@pytest.mark.slow
def test_decode_totality():
    e = _env(n=256)
    base = oracle.canon_fields(e.get_state(0))["mem"]
    bad = []
    for hi in range(256):
        for lo in range(256):
            m = base.copy()
            m[0x300], m[0x301] = hi, lo
            e.set_state(lo, canon(PC=0x300, SP=1, stack=[0x400] + [0] * 15, I=0x500, mem=m))
        for lo in range(256):
            e.run_cycles(lo, 1, 0x1)
            w = hi << 8 | lo
            if bool(e.get_state(lo)[23] & 1) == _valid_word(w):
                bad.append(w)
    assert not bad, [hex(w) for w in bad[:10]]


# ---------------------------------------------------------------- stack depth
def test_sixteen_calls_ok_seventeenth_halts():
    # 2202: call self-next repeatedly -> each call pushes; depth 16 OK, 17th halts
    rom = bytes([0x22, 0x02] * 17)
    e = _env(rom)
    e.run_cycles(0, 16)
    f = oracle.canon_fields(e.get_state(0))
    assert f["SP"] == 16 and not f["halted"]
    e.run_cycles(0, 1)
    assert oracle.canon_fields(e.get_state(0))["halted"] == 1


# ---------------------------------------------------------------- DXYN
def _draw_env(sprite: bytes, quirks=0):
    # sprite data at 0x300; program at 0x200: D12n ; 1202
    return _env(bytes([0x12, 0x00]), quirks=quirks), sprite


def _draw(e, x, y, sprite, display=None, quirks_env=None):
    f = oracle.canon_fields(e.get_state(0))
    mem = f["mem"]
    mem[0x300:0x300 + len(sprite)] = np.frombuffer(sprite, np.uint8)
    mem[0x200], mem[0x201] = 0xD1, 0x20 | len(sprite)
    V = [0] * 16
    V[1], V[2] = x, y
    disp = f["display"] if display is None else display
    e.set_state(0, canon(V=V, I=0x300, PC=0x200, mem=mem, display=disp))
    e.run_cycles(0, 1)
    f = oracle.canon_fields(e.get_state(0))
    return f["display"], f["V"][15]


def test_draw_clip_and_wrap_examples():
    e = _env()
    d, vf = _draw(e, 60, 0, b"\xFF", display=np.zeros(256, np.uint8))
    assert vf == 0
    assert list(d[0:8]) == [0, 0, 0, 0, 0, 0, 0, 0x0F]       # S:116 clip: columns 60-63
    assert not d[8:].any()
    e = _env(quirks=8)
    d, vf = _draw(e, 60, 0, b"\xFF", display=np.zeros(256, np.uint8))
    assert list(d[0:8]) == [0xF0, 0, 0, 0, 0, 0, 0, 0x0F]    # wrap quirk
    e = _env()
    d, _ = _draw(e, 74, 40, b"\x80", display=np.zeros(256, np.uint8))   # S:118 modulo
    bits = oracle.display_bits(d)
    assert bits[8, 10] == 1 and bits.sum() == 1


def test_draw_twice_restores_display_property():
    """drawing the same sprite twice erases it; VF=1 on the second draw iff
    at least one set sprite pixel lands on screen."""
    rng = np.random.default_rng(7)
    e = _env()
    for _ in range(300):
        disp = rng.integers(0, 256, 256, dtype=np.uint8) & rng.integers(0, 256, 256, dtype=np.uint8)
        n = int(rng.integers(0, 16))
        spr = bytes(rng.integers(0, 256, n, dtype=np.uint8)) if rng.random() < 0.9 else bytes(n)
        x, y = int(rng.integers(0, 256)), int(rng.integers(0, 256))
        d1, vf1 = _draw(e, x, y, spr, display=disp)
        d2, vf2 = _draw(e, x, y, spr, display=d1)
        assert np.array_equal(d2, disp)
        # brute force: count on-screen set pixels (clip rule)
        x0, y0 = x % 64, y % 32
        on = sum(1 for r, byte in enumerate(spr) for c in range(8)
                 if (byte >> (7 - c)) & 1 and y0 + r < 32 and x0 + c < 64)
        assert vf2 == (1 if on else 0)
        # first draw: VF=1 iff some on-screen sprite pixel hit a lit pixel (brute force)
        bits = oracle.display_bits(disp)
        hits = sum(1 for r, byte in enumerate(spr) for c in range(8)
                   if (byte >> (7 - c)) & 1 and y0 + r < 32 and x0 + c < 64 and bits[y0 + r, x0 + c])
        assert vf1 == (1 if hits else 0)


def _golden_font():
    rows = [line.split() for line in golden_lines("font.txt")]
    assert [int(r[0], 16) for r in rows] == list(range(16))
    return bytes(int(b, 16) for r in rows for b in r[1:])


def test_font_bytes_golden():
    """All 80 font bytes at 0x050..0x09F equal SURVEY App. B (tests/golden/font.txt), so a
    one-nibble typo in any glyph row of the oracle's table fails (A23)."""
    font = _golden_font()
    assert len(font) == 80 and font[0] == 0xF0
    f = oracle.canon_fields(_env().get_state(0))
    assert bytes(f["mem"][0x50:0xA0]) == font
    # FX29 addresses glyph VX & 15 at 0x50 + 5 * digit (App. A.4 / SURVEY App. A), and
    # drawing it renders exactly the golden rows
    e = _env()
    for k in range(16):
        mem = oracle.canon_fields(e.get_state(0))["mem"]
        mem[0x200:0x206] = [0xF3, 0x29, 0xD1, 0x25, 0x12, 0x04]
        V = [0] * 16
        V[1], V[2], V[3] = 0, 0, 0x10 | k                  # high nibble ignored
        e.set_state(0, canon(V=V, PC=0x200, mem=mem))
        e.run_cycles(0, 2)
        g = oracle.canon_fields(e.get_state(0))
        assert g["I"] == 0x50 + 5 * k
        assert bytes(g["display"].reshape(32, 8)[0:5, 0]) == font[5 * k:5 * k + 5]


def test_font_glyph_render_matches_font_bytes():
    e = _env()
    for k in range(16):
        f = oracle.canon_fields(e.get_state(0))
        mem = f["mem"]
        mem[0x200:0x206] = [0xF3, 0x29, 0xD1, 0x25, 0x12, 0x04]  # LD F,V3 ; DRW V1,V2,5
        V = [0] * 16
        V[1], V[2], V[3] = 8, 3, k
        e.set_state(0, canon(V=V, PC=0x200, mem=mem))
        e.run_cycles(0, 2)
        d = oracle.canon_fields(e.get_state(0))["display"].reshape(32, 8)
        assert list(d[3:8, 1]) == list(mem[0x50 + 5 * k:0x55 + 5 * k])


# ---------------------------------------------------------------- timers / frames
def test_timer_frame_accounting():
    e = _env(frame_skip=4)
    f = oracle.canon_fields(e.get_state(0))
    e.set_state(0, canon(PC=0x200, DT=200, ST=9, mem=f["mem"]))
    for k in range(1, 11):
        e.step(np.zeros(1, np.int32))
        f = oracle.canon_fields(e.get_state(0))
        assert f["DT"] == 200 - 4 * k                # k steps -> 4k decrements
        assert f["ST"] == max(0, 9 - 4 * k)          # saturating at 0
    e.run_frames(0, 1)
    assert oracle.canon_fields(e.get_state(0))["DT"] == 200 - 41


def test_halted_machine_is_inert():
    e = _env(bytes([0xFF, 0xFF]))   # invalid word: halts on first cycle
    f = oracle.canon_fields(e.get_state(0))
    e.set_state(0, canon(PC=0x200, DT=50, mem=f["mem"]))
    e.run_frames(0, 3)
    f = oracle.canon_fields(e.get_state(0))
    assert f["halted"] == 1 and f["DT"] == 50 and f["PC"] == 0x202


# ---------------------------------------------------------------- expressions
def test_pong_formula_bruteforce():
    """P:152 score = (V[14] // 10) - (V[14] % 10), digits by string brute force."""
    for v in range(100):
        s = f"{v:02d}"
        want = (int(s[0]) - int(s[1])) & 0xFFFFFFFF
        c = canon(V=[0] * 14 + [v, 0])
        assert oracle.eval_expr("(V14 // 10) - (V14 % 10)", c) == want
        assert oracle.eval_expr("(V[14] // 10) - (V[14] % 10)", c) == want
    assert oracle.eval_expr("(V14 // 10) - (V14 % 10)", canon(V=[0] * 14 + [42, 0])) == 2


def test_space_flight_truth_table():
    """P:154 terminated = (V[9] == 0) | (V[12] >= 0x3E)."""
    for v9 in (0, 1):
        for v12 in (0x3D, 0x3E, 0xFF):
            V = [0] * 16
            V[9], V[12] = v9, v12
            want = 1 if (v9 == 0 or v12 >= 0x3E) else 0
            assert oracle.eval_expr("(V9 == 0) | (V12 >= 0x3E)", canon(V=V)) == want


@pytest.mark.parametrize("expr,V,want", [
    ("V5", {5: 7}, 7), ("V14 == 0", {14: 0}, 1), ("V14 == 0", {14: 3}, 0),  # P:152-154 Brix
    ("V1 == 2", {1: 2}, 1), ("V1 == 2", {1: 1}, 0),                        # P:154 Tetris
    ("V2", {2: 10}, 10), ("V3 == 1", {3: 1}, 1),
    ("1 + 2 * 3", {}, 7), ("(1 + 2) * 3", {}, 9), ("10 - 4 - 3", {}, 3),
    ("1 << 2 + 1", {}, 8), ("1 | 2 ^ 3 & 4", {}, 3), ("3 > 2 == 1", {}, 1),
    ("5 / 0", {}, 0), ("7 % 0", {}, 0), ("0 - 1", {}, 0xFFFFFFFF), ("-1", {}, 0xFFFFFFFF),
    ("!0", {}, 1), ("!5", {}, 0), ("~0", {}, 0xFFFFFFFF), ("2 && 3", {}, 1), ("0 || 0", {}, 0),
    ("1 << 32", {}, 0), ("0x10 >> 4", {}, 1), ("mem[0x1050]", {}, 0xF0), ("memory[0x50]", {}, 0xF0),
    ("VA + vb + V[15]", {10: 1, 11: 2, 15: 4}, 7), ("7 // 2", {}, 3), ("0xFFFFFFFF + 1", {}, 0),
])
def test_expression_cases(expr, V, want):
    v = [0] * 16
    for k, x in V.items():
        v[k] = x
    e = _env()
    base = oracle.canon_fields(e.get_state(0))["mem"]
    assert oracle.eval_expr(expr, canon(V=v, mem=base)) == want


def test_expression_i_dt_st():
    c = canon(I=0x123, DT=5, ST=6)
    assert oracle.eval_expr("I + DT * ST", c) == 0x123 + 30


@pytest.mark.parametrize("expr,offset", [("V9 == )", 6), ("V16", 0), ("(V1", 3), ("1 +", 3),
                                          ("V1 V2", 3), ("mem[1", 5), ("", 0)])
def test_expression_syntax_errors(expr, offset):
    assert oracle.expr_error_offset(expr) == offset   # S:268 "V9 == )" -> offset 6


# ---------------------------------------------------------------- env semantics
def test_reset_obs_planes_and_first_step():
    rom, spec = workloads.game("pong_standin")
    e = oracle.OracleEnv(rom, spec, 3, 5)
    obs0 = e.reset(5).reshape(3, 4, 256)
    for j in range(3):
        for p in range(1, 4):
            assert np.array_equal(obs0[j, 0], obs0[j, p])
        f = oracle.canon_fields(e.get_state(j))
        assert np.array_equal(obs0[j, 3], f["display"])
    obs1 = e.step(np.array([0, 1, 2], np.int32))[0].reshape(3, 4, 256)
    for j in range(3):
        for p in range(0, 3):
            assert np.array_equal(obs1[j, p], obs0[j, 3])
        assert np.array_equal(obs1[j, 3], oracle.canon_fields(e.get_state(j))["display"])


def test_bool_xmajor_is_transpose_of_packed():
    rom, spec = workloads.game("brix_standin")
    a = oracle.OracleEnv(rom, spec, 2, 3)
    b = oracle.OracleEnv(rom, dict(spec, obs_format=1), 2, 3)
    for t in range(20):
        act = workloads.gen.actions(3, t, 2, 3)
        pa = a.step(act)[0].reshape(2, 4, 32, 8)
        pb = b.step(act)[0].reshape(2, 4, 64, 32)
        bits = np.unpackbits(pa, axis=3).reshape(2, 4, 32, 64)
        assert np.array_equal(bits.transpose(0, 1, 3, 2), pb)       # P:146 (4, 64, 32)


def test_telescoping_rewards_and_stats():
    """within an episode sum(reward) = final - initial score (signed);
    stats.returns = sum of ep_ret over finished episodes; integer exact."""
    rom, spec = workloads.game("brix_standin")
    n = 16
    e = oracle.OracleEnv(rom, spec, n, 11)
    ep_sum = np.zeros(n, np.int64)
    finished = 0
    total = 0
    for t in range(400):
        _, r, d, term, trunc = e.step(workloads.gen.actions(11, t, n, 3))
        ep_sum += r.astype(np.int64)
        for j in np.nonzero(d)[0]:
            total += ep_sum[j]
            ep_sum[j] = 0
            finished += 1
        for j in range(n):
            f = oracle.canon_fields(e.get_state(j))
            assert f["ep_ret"] == ep_sum[j]
    stats, _ = e.stats()
    assert stats[1] == finished and finished > 0
    assert stats[0] == total and stats[2] == n * 400


def test_out_of_range_action_is_noop_and_sticky():
    rom, spec = workloads.game("pong_standin")
    a = oracle.OracleEnv(rom, spec, 2, 1)
    b = oracle.OracleEnv(rom, spec, 2, 1)
    oa = a.step(np.array([7, -1], np.int32))
    ob = b.step(np.array([0, 0], np.int32))
    assert np.array_equal(oa[0], ob[0])
    _, rc = a.stats()
    assert rc == -8
    assert b.stats()[1] == 0


def test_determinism_and_shard_invariance():
    """A13: trajectories depend on the global env id only -> identical for any sharding."""
    rom, spec = workloads.game("pong_standin")
    full = oracle.OracleEnv(rom, spec, 8, 99, 0)
    lo = oracle.OracleEnv(rom, spec, 4, 99, 0)
    hi = oracle.OracleEnv(rom, spec, 4, 99, 4)
    for t in range(60):
        a = workloads.gen.actions(99, t, 8, 3)
        o = full.step(a)[0]
        assert np.array_equal(o[:4], lo.step(a[:4])[0])
        assert np.array_equal(o[4:], hi.step(a[4:])[0])
    for j in range(8):
        ref = full.get_state(j)
        got = lo.get_state(j) if j < 4 else hi.get_state(j - 4)
        assert np.array_equal(ref, got)


def test_truncation_and_startup():
    rom, spec = workloads.game("pong_standin", max_episode_steps=5, startup=[(0x2, 3), (0, 2)])
    e = oracle.OracleEnv(rom, spec, 1, 1)
    f = oracle.canon_fields(e.get_state(0))
    assert f["steps"] == 0
    for t in range(5):
        _, _, d, term, trunc = e.step(np.zeros(1, np.int32))
    assert d[0] == 1 and trunc[0] == 1 and term[0] == 0
    f = oracle.canon_fields(e.get_state(0))
    assert f["episode"] == 1 and f["steps"] == 0


def test_startup_runs_frames_with_keys_and_timers():
    # program: F10A (wait key -> V1) ; F215 (DT := V2) ; 1204
    rom = bytes([0xF1, 0x0A, 0xF2, 0x15, 0x12, 0x04])
    e = oracle.OracleEnv(rom, dict(BASE_SPEC, startup=[(1 << 9, 1)]), 1, 0)
    f = oracle.canon_fields(e.get_state(0))
    assert f["V"][1] == 9 and f["PC"] == 0x204


def test_halt_terminates_and_resets_same_step():
    rom = bytes([0x60, 0x05, 0xFF, 0xFF])   # V0 := 5 ; invalid -> halt
    e = _env(rom)
    _, r, d, term, trunc = e.step(np.zeros(1, np.int32))
    assert d[0] == 1 and term[0] == 1
    f = oracle.canon_fields(e.get_state(0))
    assert f["episode"] == 1 and f["PC"] == 0x200 and not f["halted"] and f["V"][0] == 0


# ---------------------------------------------------------------- coverage ROM
def test_coverage_rom_self_checks_pass():
    """c.4: all hand-derived self-test groups pass -> pass count and bitmap."""
    rom, n_groups = workloads.coverage_rom.build()
    _, spec = workloads.game("coverage")
    e = oracle.OracleEnv(rom, spec, 1, workloads.ENV_SEED)
    acts = workloads.gen.action_stream(1, 1000, 1, 17)
    total = 0.0
    for t in range(1000):
        total += float(e.step(acts[t])[1][0])
    f = oracle.canon_fields(e.get_state(0))
    assert f["mem"][0xF00] == n_groups == 20
    assert np.all(f["mem"][0xF01:0xF01 + n_groups] == 0xA5)
    assert total == n_groups                        # telescoping: score went 0 -> 20


# ---------------------------------------------------------------- intra-step frame stacking
@pytest.mark.parametrize("fs", [1, 2, 4, 6])
@pytest.mark.parametrize("game", ["pong_standin", "target_shooter_level1"])
def test_stack_frames_equals_fs1_step_end_stack(game, fs):
    """OBS_STACK_FRAMES (SPEC S:434 alternative) pinned to the default A3 stack of a
    frame_skip=1 env holding each action for fs steps: frames [t*fs+1 .. (t+1)*fs]
    are the last fs step-end displays there (planes before the step repeat the
    step-start display when fs < 4)."""
    rom, spec = workloads.game(game, terminated="0", max_episode_steps=0)
    n = 6
    a = oracle.OracleEnv(rom, dict(spec, frame_skip=fs, obs_format=16), n, 5)
    b = oracle.OracleEnv(rom, dict(spec, frame_skip=1, obs_format=0), n, 5)
    na = len(spec["action_keys"]) + 1
    for t in range(25):
        acts = workloads.gen.actions(3, t, n, na)
        oa = a.step(acts)[0].reshape(n, 4, 32, 8)
        for _ in range(fs):
            ob = b.step(acts)[0].reshape(n, 4, 32, 8)
        k = min(fs, 4)
        assert np.array_equal(oa[:, 4 - k:], ob[:, 4 - k:])
        for p in range(4 - k):                       # step-start display repeated
            assert np.array_equal(oa[:, p], ob[:, 3 - k])


def test_stack_frames_bool_layout_and_reset():
    """Flag composes with the bool layout (bit 0); a terminal step's obs is the reset
    display in all 4 planes; final_obs keeps the terminal step's frames."""
    rom, spec = workloads.game("brix_standin", max_episode_steps=7)
    n = 4
    a = oracle.OracleEnv(rom, dict(spec, obs_format=17), n, 2)
    p = oracle.OracleEnv(rom, dict(spec, obs_format=16), n, 2)
    assert a.obs_per_env == 8192 and p.obs_per_env == 1024
    for t in range(7):
        acts = workloads.gen.actions(4, t, n, 3)
        oa, _, da, _, _, fa, _, _ = a.step_ex(acts)
        op, _, dp, _, _, fp, _, _ = p.step_ex(acts)
        bits = oa.reshape(n, 4, 64, 32).transpose(0, 1, 3, 2)
        assert np.array_equal(np.packbits(bits, axis=-1).reshape(n, -1), op)
    assert da.all() and dp.all()
    op4 = op.reshape(n, 4, 256)
    assert all(np.array_equal(op4[:, 0], op4[:, q]) for q in range(1, 4))
    assert not np.array_equal(fp.reshape(n, 4, 256)[:, 3], op4[:, 3])
