"""Self-checking opcode-coverage ROM (BASELINE.json configs[0]).

The ROM runs one self-test group per opcode family.  Each group compares its
results against immediates that were worked out BY HAND from the CHIP-8
definition (Appendix A of PAPER.md, plus the readings in
DESIGN.md) -- never by running an implementation.  A group that passes
writes 0xA5 to mem[0xF00 + g] and increments the pass counter mem[0xF00].
The expected final RAM bytes are therefore known independently of any
interpreter: mem[0xF00] = N_GROUPS and mem[0xF01 .. 0xF00+N_GROUPS] = 0xA5.

After the self-tests a main loop runs forever: it polls keys (EX9E / EXA1 /
FX0A) against the action stream, draws at CXNN coordinates, exercises FX33
and folds everything into a checksum register pair (VD:VE).  That part is
pinned only by GPU<->oracle parity.

Action set: keys 0..F (17 actions, action 0 = no-op).
"""
from __future__ import annotations

from .chip8asm import assemble

PASS_BASE = 0xF00
PASS_MAGIC = 0xA5


def _chk(reg: str, val: int, fail: str) -> str:
    return f"  SE {reg}, {val}\n  JP {fail}\n"


def source() -> tuple[str, int]:
    g = []  # (name, body) ; body must fall through on success, jump to fail_<n> on failure

    # 1: 8XY4 add with carry -- hand: 200+100=300 -> 44, VF=1 ; 255+1 -> 0, VF=1 ; 1+2 -> 3, VF=0
    g.append("""
  LD V1, 200
  LD V2, 100
  ADD V1, V2
""" + _chk("V1", 44, "@F") + _chk("VF", 1, "@F") + """
  LD V1, 255
  LD V2, 1
  ADD V1, V2
""" + _chk("V1", 0, "@F") + _chk("VF", 1, "@F") + """
  LD V1, 1
  LD V2, 2
  ADD V1, V2
""" + _chk("V1", 3, "@F") + _chk("VF", 0, "@F"))

    # 2: 8XY5 VX-VY, VF = VX>=VY -- (10,5)->(5,1) (5,10)->(251,0) (7,7)->(0,1)
    g.append("""
  LD V1, 10
  LD V2, 5
  SUB V1, V2
""" + _chk("V1", 5, "@F") + _chk("VF", 1, "@F") + """
  LD V1, 5
  LD V2, 10
  SUB V1, V2
""" + _chk("V1", 251, "@F") + _chk("VF", 0, "@F") + """
  LD V1, 7
  LD V2, 7
  SUB V1, V2
""" + _chk("V1", 0, "@F") + _chk("VF", 1, "@F") + """
  LD V1, 7
  SUB V1, V1
""" + _chk("V1", 0, "@F") + _chk("VF", 1, "@F"))

    # 3: 8XY7 VY-VX, VF = VY>=VX -- VX=10,VY=5 -> 251,0 ; VX=5,VY=10 -> 5,1
    g.append("""
  LD V1, 10
  LD V2, 5
  SUBN V1, V2
""" + _chk("V1", 251, "@F") + _chk("VF", 0, "@F") + """
  LD V1, 5
  LD V2, 10
  SUBN V1, V2
""" + _chk("V1", 5, "@F") + _chk("VF", 1, "@F"))

    # 4: 8XY6 (modern: shifts VX, VY untouched) -- 0x81 -> 0x40,1 ; 0x02 -> 0x01,0
    g.append("""
  LD V1, 0x81
  LD V2, 0xFF
  SHR V1, V2
""" + _chk("V1", 0x40, "@F") + _chk("VF", 1, "@F") + _chk("V2", 0xFF, "@F") + """
  LD V1, 0x02
  SHR V1, V2
""" + _chk("V1", 0x01, "@F") + _chk("VF", 0, "@F"))

    # 5: 8XYE -- 0x81 -> 0x02,1 ; 0x40 -> 0x80,0
    g.append("""
  LD V1, 0x81
  LD V2, 0x00
  SHL V1, V2
""" + _chk("V1", 0x02, "@F") + _chk("VF", 1, "@F") + """
  LD V1, 0x40
  SHL V1, V2
""" + _chk("V1", 0x80, "@F") + _chk("VF", 0, "@F"))

    # 6: X = F, flag written last (A15) -- VF=200,V1=100: 8F14 -> VF=1 ;
    #    VF=5,V1=10: 8F15 -> VF=0 ; VF=10,V1=5: 8F15 -> VF=1 ; VF=0x81: 8FFE -> 1 ; VF=0x02: 8FF6 -> 0
    g.append("""
  LD VF, 200
  LD V1, 100
  ADD VF, V1
""" + _chk("VF", 1, "@F") + """
  LD VF, 5
  LD V1, 10
  SUB VF, V1
""" + _chk("VF", 0, "@F") + """
  LD VF, 10
  LD V1, 5
  SUB VF, V1
""" + _chk("VF", 1, "@F") + """
  LD VF, 0x81
  SHL VF, VF
""" + _chk("VF", 1, "@F") + """
  LD VF, 0x02
  SHR VF, VF
""" + _chk("VF", 0, "@F"))

    # 7: 8XY0-3, VF untouched (modern) -- F0|0F=FF ; F0&3C=30 ; F0^3C=CC ; LD V1,V2 = 3C
    g.append("""
  LD VF, 0x77
  LD V1, 0xF0
  LD V2, 0x0F
  OR V1, V2
""" + _chk("V1", 0xFF, "@F") + _chk("VF", 0x77, "@F") + """
  LD V1, 0xF0
  LD V2, 0x3C
  AND V1, V2
""" + _chk("V1", 0x30, "@F") + """
  LD V1, 0xF0
  XOR V1, V2
""" + _chk("V1", 0xCC, "@F") + """
  LD V1, V2
""" + _chk("V1", 0x3C, "@F") + _chk("VF", 0x77, "@F"))

    # 8: skips taken / not taken (3XNN 4XNN 5XY0 9XY0)
    g.append("""
  LD V1, 5
  LD V2, 5
  LD V3, 6
  SE V1, 5
  JP @F
  SE V1, 6
  JP @L1
  JP @F
@L1:
  SNE V1, 6
  JP @F
  SNE V1, 5
  JP @L2
  JP @F
@L2:
  SE V1, V2
  JP @F
  SE V1, V3
  JP @L3
  JP @F
@L3:
  SNE V1, V3
  JP @F
  SNE V1, V2
  JP @L4
  JP @F
@L4:
""")

    # 9: nested CALL / RET -- V5 counts 3 increments, returns in order
    g.append("""
  LD V5, 0
  CALL sub_a
""" + _chk("V5", 3, "@F"))

    # 10: BNNN = NNN + V0 -- V0=4 -> jt+4
    g.append("""
  LD V0, 4
  JP V0, @JT
@JT:
  JP @F
  JP @F
  JP @OK
@OK:
""")

    # 11: FX1E (16-bit, VF untouched), FX55/FX65 with (I+k)&0xFFF (A18)
    #     I=0xE00+0x10 -> 0xE10 ; I=0xFFF+2 -> 0x1001 -> address 0x001
    g.append("""
  LD VF, 0x42
  LD I, 0xE00
  LD V1, 0x10
  ADD I, V1
""" + _chk("VF", 0x42, "@F") + """
  LD V0, 0x5A
  LD [I], V0
  LD I, 0xE10
  LD V0, 0
  LD V0, [I]
""" + _chk("V0", 0x5A, "@F") + """
  LD I, 0xFFF
  LD V1, 2
  ADD I, V1
  LD V0, 0x6B
  LD [I], V0
  LD I, 0x001
  LD V0, 0
  LD V0, [I]
""" + _chk("V0", 0x6B, "@F"))

    # 12: FX29 -> 0x50 + 5*(VX&F); canonical font bytes (A23)
    #     'A' at 0x82 first byte F0 ; 0x1F -> 'F' at 0x9B: F0 80 ; '1' at 0x55: 20
    g.append("""
  LD V1, 0x0A
  LD F, V1
  LD V0, [I]
""" + _chk("V0", 0xF0, "@F") + """
  LD V1, 0x1F
  LD F, V1
  LD V1, [I]
""" + _chk("V0", 0xF0, "@F") + _chk("V1", 0x80, "@F") + """
  LD V1, 0x01
  LD F, V1
  LD V0, [I]
""" + _chk("V0", 0x20, "@F"))

    # 13: FX33 BCD -- 156 -> 1,5,6 ; 0 -> 0,0,0 ; 255 -> 2,5,5
    g.append("""
  LD I, 0xE20
  LD V3, 156
  LD B, V3
  LD V2, [I]
""" + _chk("V0", 1, "@F") + _chk("V1", 5, "@F") + _chk("V2", 6, "@F") + """
  LD V3, 0
  LD B, V3
  LD V2, [I]
""" + _chk("V0", 0, "@F") + _chk("V1", 0, "@F") + _chk("V2", 0, "@F") + """
  LD V3, 255
  LD B, V3
  LD V2, [I]
""" + _chk("V0", 2, "@F") + _chk("V1", 5, "@F") + _chk("V2", 5, "@F"))

    # 14: FX55 / FX65 round trip of V0..V5, I unchanged (modern)
    g.append("""
  LD V0, 11
  LD V1, 22
  LD V2, 33
  LD V3, 44
  LD V4, 55
  LD V5, 66
  LD I, 0xE30
  LD [I], V5
  LD V0, 0
  LD V1, 0
  LD V2, 0
  LD V3, 0
  LD V4, 0
  LD V5, 0
  LD V5, [I]
""" + "".join(_chk(f"V{k}", 11 * (k + 1), "@F") for k in range(6)) + """
  LD V0, 0
  LD V0, [I]
""" + _chk("V0", 11, "@F"))

    # 15: DXYN -- XOR double draw, clipping, modulo start, DXY0, VF as coordinate
    g.append("""
  CLS
  LD I, spr2
  LD V1, 10
  LD V2, 10
  DRW V1, V2, 2
""" + _chk("VF", 0, "@F") + """
  DRW V1, V2, 2
""" + _chk("VF", 1, "@F") + """
  DRW V1, V2, 2
""" + _chk("VF", 0, "@F") + """
  DRW V1, V2, 2
""" + _chk("VF", 1, "@F") + """
  LD I, spr_ff
  LD V1, 60
  LD V2, 0
  DRW V1, V2, 1
""" + _chk("VF", 0, "@F") + """
  LD I, spr_dot
  LD V1, 63
  DRW V1, V2, 1
""" + _chk("VF", 1, "@F") + """
  DRW V1, V2, 1
""" + _chk("VF", 0, "@F") + """
  LD V1, 0
  DRW V1, V2, 1
""" + _chk("VF", 0, "@F") + """
  DRW V1, V2, 1
""" + _chk("VF", 1, "@F") + """
  CLS
  LD I, spr_col
  LD V1, 5
  LD V2, 31
  DRW V1, V2, 2
""" + _chk("VF", 0, "@F") + """
  LD I, spr_dot
  LD V2, 0
  DRW V1, V2, 1
""" + _chk("VF", 0, "@F") + """
  LD V2, 31
  DRW V1, V2, 1
""" + _chk("VF", 1, "@F") + """
  CLS
  LD V1, 74
  LD V2, 40
  DRW V1, V2, 1
""" + _chk("VF", 0, "@F") + """
  LD V1, 10
  LD V2, 8
  DRW V1, V2, 1
""" + _chk("VF", 1, "@F") + """
  LD VF, 1
  DRW V1, V2, 0
""" + _chk("VF", 0, "@F") + """
  LD VF, 20
  LD V1, 3
  DRW VF, V1, 1
""" + _chk("VF", 0, "@F") + """
  LD V2, 20
  DRW V2, V1, 1
""" + _chk("VF", 1, "@F") + """
  CLS
""")

    # 16: FX15 / FX07 across frames: first change 200 -> 199 ; DT saturates at 0
    g.append("""
  LD V1, 200
  LD DT, V1
@W1:
  LD V2, DT
  SNE V2, 200
  JP @W1
""" + _chk("V2", 199, "@F") + """
  LD V1, 1
  LD DT, V1
@W2:
  LD V2, DT
  SE V2, 0
  JP @W2
  LD V3, 40
@W3:
  ADD V3, 255
  SE V3, 0
  JP @W3
  LD V2, DT
""" + _chk("V2", 0, "@F"))

    # 17: CXNN with NN=0 is 0; NN=0x0F keeps only the low nibble
    g.append("""
  LD V1, 0x55
  RND V1, 0
""" + _chk("V1", 0, "@F") + """
  RND V2, 0x0F
  LD V4, 0xF0
  AND V2, V4
""" + _chk("V2", 0, "@F"))

    # 18: 7XNN wraps mod 256 and leaves VF -- 0xFF+1 -> 0 ; VF stays 0x33
    g.append("""
  LD VF, 0x33
  LD V1, 0xFF
  ADD V1, 1
""" + _chk("V1", 0, "@F") + _chk("VF", 0x33, "@F") + """
  ADD V1, 0xFF
""" + _chk("V1", 0xFF, "@F"))

    # 19: self-modifying code: FX55 rewrites the next instruction 6300 -> 632A
    g.append("""
  LD I, @SMC
  LD V0, 0x63
  LD V1, 0x2A
  LD [I], V1
  LD V3, 0
@SMC:
  LD V3, 0
""" + _chk("V3", 0x2A, "@F"))

    # 20: odd PC -- jump into an odd address and execute from there
    g.append("""
  LD V1, 0
  JP @ODD
  .db 0x12
@ODD:
  LD V1, 0x77
""" + _chk("V1", 0x77, "@F"))

    # ---------------------------------------------------------------- assemble
    n = len(g)
    out = [f"; generated by workloads/coverage_rom.py -- {n} self-test groups",
           "  JP start", "start:"]
    for i, body in enumerate(g, 1):
        b = body.replace("@F", f"fail_{i}").replace("@", f"g{i}_")
        out.append(f"; ---- group {i}")
        out.append(b)
        out.append(f"  LD V0, {i}\n  CALL mark\nfail_{i}:")
    out.append("""
; ---- main loop (parity-only region)
  LD VD, 0
  LD VE, 0
  LD V6, 0
loop:
  ADD V6, 1
  LD V7, 0x0F
  AND V6, V7
  SKNP V6
  ADD VE, 3
  SKP V6
  ADD VE, 5
  RND V8, 0x3F
  RND V9, 0x1F
  LD I, spr3
  DRW V8, V9, 3
  ADD VE, VF
  ADD VD, VF
  LD I, 0xF40
  LD B, VE
  LD V2, [I]
  ADD VD, V2
  LD I, 0xF43
  LD [I], V9
  SE V6, 0
  JP loop
  LD VA, K
  ADD VE, VA
  LD V1, 7
  LD ST, V1
  LD DT, V1
  JP loop

mark:            ; V0 = group number
  LD I, 0xF00
  ADD I, V0
  LD V0, 0xA5
  LD [I], V0
  LD I, 0xF00
  LD V0, [I]
  ADD V0, 1
  LD [I], V0
  RET

sub_a:
  ADD V5, 1
  CALL sub_b
  ADD V5, 1
  RET
sub_b:
  ADD V5, 1
  RET

spr2:   .db 0b11000011, 0b00111100
spr_ff: .db 0xFF
spr_dot: .db 0x80
spr_col: .db 0x80, 0x80
spr3:   .db 0b10100000, 0b01000000, 0b10100000
""")
    return "\n".join(out), n


def build() -> tuple[bytes, int]:
    text, n = source()
    rom, _ = assemble(text)
    return rom, n


SPEC = {
    # SURVEY c.4: score = pass count, no termination, keys 0..F (17 actions)
    "score": "mem[0xF00]",
    "terminated": "0",
    "action_keys": list(range(16)),
    "frame_skip": 4,
    "instructions_per_frame": 12,
    "max_episode_steps": 0,
}
