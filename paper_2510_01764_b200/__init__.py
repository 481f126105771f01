"""B200-native batched Octax (arXiv 2510.01764) environment step.

The hot path -- N CHIP-8 VMs stepped in lockstep with frame skip, DXYN XOR
drawing, timers, reward / termination, stacked observations and auto-reset --
is hand-written CUDA for sm_100a in ``csrc/`` behind the C ABI of
``include/octax.h``; ``octax.py`` is a thin ctypes binding.
"""
from .octax import OctaxEnv, OctaxError, load_library, SYMBOLS  # noqa: F401
