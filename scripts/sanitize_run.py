#!/usr/bin/env python
"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
exercises every kernel (step, reset, bool-obs expansion, action generator,
get/set state) on a few hundred envs including ragged CTAs, quirks, dirty-RAM
fetches, startup segments and the cooperative DXYN path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2510_01764_b200 import OctaxEnv  # noqa: E402


def run(rom, spec, n, steps, seed=1):
    e = OctaxEnv(rom, spec, n, seed)
    a = torch.empty(n, dtype=torch.int32, device="cuda")
    for t in range(steps):
        e.gen_actions(seed, t, a)
        e.step(a)
    e.reset(seed + 1)
    s = e.get_states([0, n - 1])
    e.set_state(n - 1, s[0])
    e.step(a)
    torch.cuda.synchronize()
    e.close()


def main():
    rom, spec = workloads.game("coverage")
    run(rom, spec, 1, 60)
    rom, spec = workloads.game("brix_standin", obs_format=1, startup=[(1 << 4, 3)], max_episode_steps=17)
    run(rom, spec, 257, 40)
    for q in (0, 31):
        rom = workloads.gen.fuzz_rom(5 + q, n_instr=300)
        spec = dict(workloads.DEFAULTS, score="V0 + mem[I]", terminated="VE == 3", action_keys=list(range(16)),
                    quirks=q, max_episode_steps=25)
        run(rom, spec, 300, 40)
    # a sprite-heavy ROM: 15-row sprites from many lanes -> cooperative DXYN path
    big = workloads.chip8asm.assemble("""
        LD I, spr
    loop:
        RND V1, 0x3F
        RND V2, 0x1F
        DRW V1, V2, 15
        JP loop
    spr: .fill 15, 0xFF
    """)[0]
    spec = dict(workloads.DEFAULTS, score="VF", terminated="0", action_keys=[1])
    run(big, spec, 200, 20)
    rom, spec = workloads.game("target_shooter_level3")
    run(rom, spec, 129, 40)
    print("sanitize_run: OK")


if __name__ == "__main__":
    main()
