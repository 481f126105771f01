"""NEXT-4 ROM tooling (-m "not gpu"): the static key-operand scan recovers the
paper's own Target Shooter action set from the assembled listing, and
the FX33 scan finds the BCD-displayed registers."""
from __future__ import annotations

import workloads
from paper_2510_01764_b200 import romtools


def test_mnemonics_cover_the_isa():
    assert romtools.mnemonic(0x00E0) == "CLS" and romtools.mnemonic(0x00EE) == "RET"
    assert romtools.mnemonic(0xD015) == "DRW V0, V1, 5"
    assert romtools.mnemonic(0xF533) == "LD B, V5"
    assert romtools.mnemonic(0xFFFF) == "DW 0xffff"              # S:98 invalid
    assert romtools.mnemonic(0x8126) == "SHR V1, V2"
    assert romtools.mnemonic(0xE1A1) == "SKNP V1"


def test_target_shooter_keys_match_paper_action_set():
    for lvl in (1, 2, 3):
        rom, spec = workloads.game(f"target_shooter_level{lvl}")
        facts = romtools.analyse(rom)
        assert sorted(facts.keys) == sorted(spec["action_keys"]) == [5, 6, 7, 8, 9]
        assert facts.uses_random and facts.draws >= 4


def test_bcd_scan_and_reachability():
    rom, _ = workloads.game("coverage")
    facts = romtools.analyse(rom)
    assert facts.bcd_registers == [0x3, 0xE]      # LD B, V3 (self-tests) ; LD B, VE (main loop)
    code = romtools.disassemble(rom)
    addrs = [a for a, _, _ in code]
    assert addrs[0] == 0x200 and len(addrs) == len(set(addrs))
    # the sprite data at the end of the ROM is not reached as code
    _, syms = workloads.chip8asm.assemble(workloads.coverage_rom.source()[0])
    assert syms["spr2"] not in addrs


def test_suggest_spec_labels_provenance():
    rom, _ = workloads.game("pong_standin")
    s = romtools.suggest_spec(rom)
    assert sorted(s["action_keys"]) == [1, 4]      # == the paper's Pong keys
    assert "not from paper" in s["provenance"]
