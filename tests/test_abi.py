"""C-ABI library checks that need no GPU (-m "not gpu"): the in-tree
liboctax.so builds for sm_100a, loads, exports every symbol include/octax.h
declares, contains sm_100a SASS with the TMA bulk copy, and rejects bad input
on the host path without touching a device."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2510_01764_b200 import build
    build.build()
    from paper_2510_01764_b200 import octax
    return octax.load_library()


def _declared():
    src = open(os.path.join(ROOT, "include", "octax.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(octax_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported(lib):
    names = _declared()
    assert len(names) >= 13
    for n in names:
        assert hasattr(lib, n), n
    from paper_2510_01764_b200.octax import SYMBOLS
    assert sorted(SYMBOLS) == names


def test_checked_build_exports_same_symbols(lib):
    from paper_2510_01764_b200 import build
    so = build.build(checked=True)
    L = ctypes.CDLL(so)
    for n in _declared():
        assert hasattr(L, n), n


def test_sass_is_sm100a_with_bulk_copy(lib):
    so = os.path.join(ROOT, "paper_2510_01764_b200", "liboctax.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "UBLKCP" in out          # cp.async.bulk (TMA bulk copy) of the ROM image
    assert "SYNCS" in out           # mbarrier


def _spec(**over):
    from paper_2510_01764_b200.octax import _make_spec
    s = {"score": "V5", "terminated": "V14 == 0", "action_keys": [1, 4]}
    s.update(over)
    return _make_spec(s)


@pytest.mark.parametrize("rom_len,over,code", [
    (0, {}, -2), (3585, {}, -3), (2, {"action_keys": [1, 1]}, -4), (2, {"action_keys": [16]}, -4),
    (2, {"frame_skip": 0}, -4), (2, {"instructions_per_frame": 0}, -4), (2, {"quirks": 64}, -4),
    (2, {"score": "V9 == )"}, -5), (2, {"terminated": "V16"}, -5), (2, {"obs_format": 3}, -4),
    (2, {"score": "(" * 9 + "1" + ")" * 9 + "+" + "+".join(["(1+(1+(1+(1+(1+(1+(1+(1+1)))))))))"])}, -5),
])
def test_create_rejects_bad_input_on_host(lib, rom_len, over, code):
    from paper_2510_01764_b200.octax import _Opts
    cs, keep = _spec(**over)
    rom = (ctypes.c_uint8 * max(1, rom_len))()
    h = ctypes.c_void_p()
    rc = lib.octax_create(rom, rom_len, ctypes.byref(cs), 4, 1, None, ctypes.byref(h))
    assert rc == code, lib.octax_last_error()
    assert h.value is None
    msg = lib.octax_last_error().decode()
    assert msg
    if code == -5 and "V9" in str(over):
        assert "at byte 6" in msg      # S:268 "V9 == )" -> offset 6


def test_null_arguments(lib):
    assert lib.octax_step(None, None, None, None, None, None, None) == -1
    assert lib.octax_stats(None, None) == -1
    lib.octax_destroy(None)


def test_gymnax_key_to_seed():
    """Gymnax front end: reset keys map to the uint64 seed (int, or [hi, lo] uint32 words)."""
    from paper_2510_01764_b200.gymnax_env import seed_from_key
    assert seed_from_key(7) == 7 and seed_from_key(-1) == 2**64 - 1
    assert seed_from_key([0x12345678, 0x9ABCDEF0]) == 0x123456789ABCDEF0
    with pytest.raises(ValueError):
        seed_from_key([1, 2, 3])


def test_create_rejects_empty_and_oversized_batches(lib):
    """n_envs = 0 and n_envs > 2^31 are refused on the host, before any device allocation."""
    cs, keep = _spec()
    rom = (ctypes.c_uint8 * 2)(0x12, 0x00)
    for n in (0, (1 << 31) + 1):
        h = ctypes.c_void_p()
        assert lib.octax_create(rom, 2, ctypes.byref(cs), n, 1, None, ctypes.byref(h)) == -1
        assert h.value is None and "n_envs" in lib.octax_last_error().decode()


def test_null_arguments_new_entry_points(lib):
    """octax_rollout / octax_step_host_frame / octax_step_host refuse NULL handles and buffers."""
    assert lib.octax_rollout(None, 4, None, 0, 0, None, 0, None, None, None, None, 0) == -1
    assert lib.octax_step_host_frame(None, None, None, None, None, None, None) == -1
    assert lib.octax_step_host(None, None, None, None, None, None, None) == -1


def test_kernel_selection_rejects_null_and_bad_values(lib):
    """octax_set_kernel / octax_get_kernel (include/octax.h): NULL handle or output refused on the
    host; the three OCTAX_KERNEL_* values are the binding's KERNELS table."""
    from paper_2510_01764_b200.octax import KERNELS
    assert lib.octax_set_kernel(None, 0) == -1
    k = ctypes.c_int(0)
    assert lib.octax_get_kernel(None, ctypes.byref(k)) == -1
    hdr = open(os.path.join(ROOT, "include", "octax.h")).read()
    for name, val in KERNELS.items():
        assert f"#define OCTAX_KERNEL_{name.upper()} {val}" in hdr
