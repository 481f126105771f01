import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, workloads, oracle
from paper_2510_01764_b200 import OctaxEnv
rom, spec = workloads.game("coverage")
g = OctaxEnv(rom, spec, 1, workloads.ENV_SEED)
o = oracle.OracleEnv(rom, spec, 1, workloads.ENV_SEED)
for t in range(3):
    a = workloads.gen.actions(1, t, 1, 17)
    g.step(torch.from_numpy(a).cuda()); o.step(a)
    fg = oracle.canon_fields(g.get_state(0)); fo = oracle.canon_fields(o.get_state(0))
    print(t, "gpu", fg["mem"][0xF00:0xF16].tolist(), "pc", hex(fg["PC"]))
    print(t, "ora", fo["mem"][0xF00:0xF16].tolist(), "pc", hex(fo["PC"]))
