"""Hand-written edge-case ROMs: the places where a fast GPU
path can silently disagree with the plain oracle.  Input generator only (ROM
bytes via the tiny assembler); both sides execute them.

Each entry: name -> (assembly source, spec overrides).
"""
from __future__ import annotations

from .chip8asm import assemble

EDGE_ROMS = {
    # FX55 overwrites the NEXT instruction (dirty-block fetch), then FX55 across a 64-B
    # block boundary, FX65 from a block dirty in some lanes only (RND decides)
    "self_modify": ("""
    start:
        LD I, target
        LD V0, 0x61
        LD V1, 0x2A
        LD [I], V1
    target:
        LD V1, 0x00
        RND V2, 1
        SE V2, 0
        JP skipwr
        LD I, 0x23E          ; 0x23E..0x241 crosses the 0x240 block boundary
        LD [I], V3
    skipwr:
        LD I, 0x23E
        LD V3, [I]
        ADD V5, V3
        LD I, 0x300
        LD B, V5
        LD V2, [I]
        ADD V6, V2
        JP start
    """, {}),
    # odd PC: jump into the middle of a word, fetch straddling a 64-B block boundary
    "odd_pc": ("""
        JP odd1
        .db 0x00
    odd1:
        LD V1, 0x11        ; at an odd address
        ADD V2, 1
        JP 0x23F           ; 0x23F..0x240 straddles blocks 8 and 9
        .org 0x23F
        .dw 0x7303         ; ADD V3, 3 at the block edge
        JP 0x201
    """, {}),
    # PC at 0xFFE executes; the next fetch at 0x1000 halts -> terminated -> same-step reset
    "pc_edge": ("""
        LD V0, 0x73
        LD V1, 0x01
        LD I, 0xFFE
        LD [I], V1
        JP 0xFFE
    """, {"terminated": "0"}),
    # address edges: FX33 at I=0xFFE wraps to 0x000; DXYN with I=0xFFC reads past 0xFFF as 0;
    # FX1E overflow past 0xFFFF
    "addr_edges": ("""
        LD V1, 123
        LD I, 0xFFE
        LD B, V1
        LD I, 0xFFC
        LD V2, 60
        LD V3, 31
        DRW V2, V3, 8
        LD V4, 0xFF
    loop:
        ADD I, V4
        ADD V5, 1
        SE V5, 0
        JP loop
        LD I, 0x000
        LD V2, [I]
        ADD V6, V0
        JP 0x200
    """, {}),
    # draw edges: x=63 / y=31 clipping, DXY0, VF as a coordinate, many lanes drawing
    # different row counts in the same cycle (RND), wrap quirk in a second spec
    "draw_edges": ("""
        LD I, spr
    loop:
        LD V1, 63
        LD V2, 31
        DRW V1, V2, 15
        DRW V1, V2, 0
        LD VF, 62
        DRW VF, V2, 3
        RND V3, 0x3F
        RND V4, 0x1F
        RND V5, 0x0F
        SE V5, 0
        DRW V3, V4, 1
        SNE V5, 7
        DRW V3, V4, 15
        SNE V5, 3
        DRW V4, V3, 9
        ADD V6, VF
        JP loop
    spr: .db 0xFF, 0x81, 0xC3, 0xE7, 0xFF, 0x00, 0x18, 0x3C, 0x7E, 0xFF, 0x01, 0x80, 0x55, 0xAA, 0xFF
    """, {}),
    # flags: 8FF4 / 8FF5 / 8FFE (X = Y = F), 8XY5 with X == Y
    "flags": ("""
    loop:
        RND VF, 0xFF
        ADD VF, VF
        ADD V1, VF
        RND VF, 0xFF
        SUB VF, VF
        ADD V1, VF
        RND VF, 0xFF
        SHL VF, VF
        ADD V1, VF
        RND V2, 0xFF
        SUB V2, V2
        ADD V1, VF
        JP loop
    """, {}),
    # control: 16 nested calls then RET x16; then the 17th call halts (in-step reset)
    "deep_calls": ("""
        LD V0, 0
        CALL f
        ADD V1, 1
        SE V1, 3
        JP 0x200
        CALL g
    f:  ADD V0, 1
        SE V0, 16
        CALL f
        RET
    g:  CALL g
    """, {"terminated": "0"}),
    # keys: FX0A on the last cycle of a frame, FX0A with no key for a whole step,
    # EX9E on VX > 15 (masked to the low nibble)
    "keys": ("""
    loop:
        LD V1, 0x1A
        SKNP V1
        ADD V2, 1
        SKP V1
        ADD V3, 1
        LD V4, K
        ADD V5, V4
        ADD V6, 1
        LD V7, DT
        SE V7, 0
        JP loop
        LD V7, 3
        LD DT, V7
        JP loop
    """, {"instructions_per_frame": 11}),
    # timers: FX15 then FX07 in the same frame and across frames, DT saturation, ST
    "timers": ("""
    loop:
        RND V1, 0x07
        LD DT, V1
        LD V2, DT
        LD ST, V1
        ADD V3, V2
        LD V4, DT
        SE V4, 0
        JP wait
        JP loop
    wait:
        LD V5, DT
        ADD V6, 1
        SE V5, 0
        JP wait
        JP loop
    """, {}),
    # RNG across resets: CXNN with NN=0 still advances the counter; lanes reset at
    # different steps (termination depends on the random byte)
    "rng_resets": ("""
        RND V1, 0x00
        RND V2, 0xFF
        RND V3, 0x0F
        ADD V4, 1
        SE V3, 5
        JP 0x202
        LD V5, 1
        JP 0x202
    """, {"terminated": "V5 == 1"}),
}


def rom(name: str) -> bytes:
    return assemble(EDGE_ROMS[name][0])[0]
