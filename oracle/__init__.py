"""Octax CPU oracle -- TEST INFRASTRUCTURE ONLY.

A ctypes binding over ``liboctax_oracle.so`` (plain single-threaded C, see
``octax_oracle.c``).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this package.  The product package ``paper_2510_01764_b200`` never imports
it, and this package never imports the product package.

Inputs are plain Python values (ROM bytes, a spec dict, numpy arrays), so the
same seeded inputs from ``workloads`` can be handed to both sides.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboctax_oracle.so")
_SRC = os.path.join(_HERE, "octax_oracle.c")

CANON_BYTES = 5200
OBS_PACKED = 0
OBS_BOOL_XMAJOR = 1


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no vectorisation flags needed)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", "-o", _SO, _SRC]
        )
    return _SO


class _Seg(ctypes.Structure):
    _fields_ = [("keymask", ctypes.c_uint16), ("frames", ctypes.c_uint32)]


class _Spec(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_uint32),
        ("score_expr", ctypes.c_char_p),
        ("terminated_expr", ctypes.c_char_p),
        ("action_keys", ctypes.POINTER(ctypes.c_uint8)),
        ("n_action_keys", ctypes.c_uint32),
        ("startup", ctypes.POINTER(_Seg)),
        ("n_startup", ctypes.c_uint32),
        ("frame_skip", ctypes.c_uint32),
        ("instructions_per_frame", ctypes.c_uint32),
        ("max_episode_steps", ctypes.c_uint32),
        ("quirks", ctypes.c_uint32),
        ("obs_format", ctypes.c_uint32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P = ctypes.c_void_p
        u8p = ctypes.POINTER(ctypes.c_uint8)
        L.octax_oracle_create.argtypes = [u8p, ctypes.c_size_t, ctypes.POINTER(_Spec),
                                          ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.POINTER(P)]
        L.octax_oracle_reset.argtypes = [P, ctypes.c_uint64, P]
        L.octax_oracle_step.argtypes = [P, P, P, P, P, P, P]
        L.octax_oracle_step_ex.argtypes = [P, P, P, P, P, P, P, P, P, P]
        L.octax_oracle_stats.argtypes = [P, P]
        L.octax_oracle_get_state.argtypes = [P, ctypes.c_uint64, P]
        L.octax_oracle_set_state.argtypes = [P, ctypes.c_uint64, P]
        L.octax_oracle_destroy.argtypes = [P]
        L.octax_oracle_destroy.restype = None
        L.octax_oracle_last_error.restype = ctypes.c_char_p
        L.octax_oracle_run_cycles.argtypes = [P, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint16]
        L.octax_oracle_run_frames.argtypes = [P, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint16]
        L.octax_oracle_eval_expr.argtypes = [ctypes.c_char_p, P, ctypes.POINTER(ctypes.c_uint32),
                                             ctypes.POINTER(ctypes.c_size_t)]
        L.octax_oracle_philox4x32_10.argtypes = [P, P, P]
        L.octax_oracle_philox4x32_10.restype = None
        L.octax_oracle_synthetic_action.argtypes = [ctypes.c_uint64, ctypes.c_uint64,
                                                    ctypes.c_uint64, ctypes.c_uint32]
        L.octax_oracle_synthetic_action.restype = ctypes.c_int32
        L.octax_oracle_counters.argtypes = [P, ctypes.c_uint64, P]
        L.octax_oracle_tick_timers.argtypes = [P, ctypes.c_uint64]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def _check(rc: int) -> None:
    if rc != 0:
        raise OracleError(rc, lib().octax_oracle_last_error().decode())


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def _make_spec(spec: dict):
    keys = bytes(spec.get("action_keys", [1]))
    keys_arr = (ctypes.c_uint8 * max(1, len(keys)))(*keys)
    segs = spec.get("startup", [])
    seg_arr = (_Seg * max(1, len(segs)))(*[_Seg(int(m), int(f)) for (m, f) in segs])
    s = _Spec()
    s.abi_version = spec.get("abi_version", 1)
    s.score_expr = spec.get("score", "0").encode() if spec.get("score") is not None else None
    s.terminated_expr = (spec.get("terminated", "0").encode()
                         if spec.get("terminated") is not None else None)
    s.action_keys = ctypes.cast(keys_arr, ctypes.POINTER(ctypes.c_uint8))
    s.n_action_keys = len(keys)
    s.startup = ctypes.cast(seg_arr, ctypes.POINTER(_Seg))
    s.n_startup = len(segs)
    s.frame_skip = spec.get("frame_skip", 4)
    s.instructions_per_frame = spec.get("instructions_per_frame", 12)
    s.max_episode_steps = spec.get("max_episode_steps", 10000)
    s.quirks = spec.get("quirks", 0)
    s.obs_format = spec.get("obs_format", OBS_PACKED)
    return s, (keys_arr, seg_arr)


class OracleEnv:
    """n independent CHIP-8 envs with global ids env_offset .. env_offset+n-1."""

    def __init__(self, rom: bytes, spec: dict, n_envs: int, seed: int, env_offset: int = 0):
        self.spec = dict(spec)
        self.n = n_envs
        self.n_actions = len(spec.get("action_keys", [1])) + 1
        self.obs_format = spec.get("obs_format", OBS_PACKED)
        self.obs_per_env = 1024 if (self.obs_format & 1) == OBS_PACKED else 8192
        cs, keep = _make_spec(spec)
        rom_arr = (ctypes.c_uint8 * max(1, len(rom)))(*rom)
        h = ctypes.c_void_p()
        _check(lib().octax_oracle_create(rom_arr, len(rom), ctypes.byref(cs), n_envs,
                                         seed & (2**64 - 1), env_offset, ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().octax_oracle_destroy(self._h)
            self._h = None

    __del__ = close

    def reset(self, seed: int) -> np.ndarray:
        obs = np.zeros((self.n, self.obs_per_env), np.uint8)
        _check(lib().octax_oracle_reset(self._h, seed & (2**64 - 1), _ptr(obs)))
        return obs

    def step(self, actions):
        a = np.ascontiguousarray(actions, dtype=np.int32)
        assert a.shape == (self.n,)
        obs = np.zeros((self.n, self.obs_per_env), np.uint8)
        rew = np.zeros(self.n, np.float32)
        done = np.zeros(self.n, np.uint8)
        term = np.zeros(self.n, np.uint8)
        trunc = np.zeros(self.n, np.uint8)
        _check(lib().octax_oracle_step(self._h, _ptr(a), _ptr(obs), _ptr(rew), _ptr(done),
                                       _ptr(term), _ptr(trunc)))
        return obs, rew, done, term, trunc

    def step_ex(self, actions):
        """Step plus extras: (obs, reward, done, term, trunc, final_obs, ep_return, ep_length)."""
        a = np.ascontiguousarray(actions, dtype=np.int32)
        obs = np.zeros((self.n, self.obs_per_env), np.uint8)
        fin = np.zeros((self.n, self.obs_per_env), np.uint8)
        rew = np.zeros(self.n, np.float32)
        done, term, trunc = (np.zeros(self.n, np.uint8) for _ in range(3))
        er = np.zeros(self.n, np.int32)
        el = np.zeros(self.n, np.uint32)
        _check(lib().octax_oracle_step_ex(self._h, _ptr(a), _ptr(obs), _ptr(rew), _ptr(done), _ptr(term),
                                          _ptr(trunc), _ptr(fin), _ptr(er), _ptr(el)))
        return obs, rew, done, term, trunc, fin, er, el

    def step_into(self, actions, obs, rew, done, term=None, trunc=None) -> None:
        """Step writing into caller-provided (preallocated) numpy buffers."""
        _check(lib().octax_oracle_step(self._h, _ptr(actions), _ptr(obs), _ptr(rew), _ptr(done),
                                       _ptr(term), _ptr(trunc)))

    def stats(self):
        out = np.zeros(4, np.int64)
        rc = lib().octax_oracle_stats(self._h, _ptr(out))
        return out, rc

    def get_state(self, env: int) -> np.ndarray:
        c = np.zeros(CANON_BYTES, np.uint8)
        _check(lib().octax_oracle_get_state(self._h, env, _ptr(c)))
        return c

    def set_state(self, env: int, canon: np.ndarray) -> None:
        c = np.ascontiguousarray(canon, dtype=np.uint8)
        assert c.shape == (CANON_BYTES,)
        _check(lib().octax_oracle_set_state(self._h, env, _ptr(c)))

    def run_cycles(self, env: int, n: int, keys: int = 0) -> None:
        _check(lib().octax_oracle_run_cycles(self._h, env, n, keys))

    def run_frames(self, env: int, n: int, keys: int = 0) -> None:
        _check(lib().octax_oracle_run_frames(self._h, env, n, keys))

    def tick_timers(self, env: int) -> None:
        _check(lib().octax_oracle_tick_timers(self._h, env))

    def counters(self, env: int) -> np.ndarray:
        out = np.zeros(17, np.uint64)
        _check(lib().octax_oracle_counters(self._h, env, _ptr(out)))
        return out


def eval_expr(expr: str, canon: np.ndarray | None = None) -> int:
    v = ctypes.c_uint32()
    off = ctypes.c_size_t()
    c = None if canon is None else np.ascontiguousarray(canon, dtype=np.uint8)
    _check(lib().octax_oracle_eval_expr(expr.encode(), _ptr(c) if c is not None else None,
                                        ctypes.byref(v), ctypes.byref(off)))
    return v.value


def expr_error_offset(expr: str) -> int | None:
    v = ctypes.c_uint32()
    off = ctypes.c_size_t()
    rc = lib().octax_oracle_eval_expr(expr.encode(), None, ctypes.byref(v), ctypes.byref(off))
    return None if rc == 0 else off.value


def philox4x32_10(ctr, key):
    c = np.array(ctr, np.uint32)
    k = np.array(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().octax_oracle_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return [int(x) for x in out]


def synthetic_action(aseed: int, t: int, gid: int, n_actions: int) -> int:
    return int(lib().octax_oracle_synthetic_action(aseed & (2**64 - 1), t, gid, n_actions))


def synthetic_actions(aseed: int, t: int, gids, n_actions: int) -> np.ndarray:
    return np.array([synthetic_action(aseed, t, int(g), n_actions) for g in gids], np.int32)


# ---- canonical-state field helpers (SURVEY c.6 layout) ----
def canon_fields(c: np.ndarray) -> dict:
    c = np.asarray(c, np.uint8)
    le16 = lambda o: int(c[o]) | (int(c[o + 1]) << 8)
    le32 = lambda o: int(c[o]) | (int(c[o + 1]) << 8) | (int(c[o + 2]) << 16) | (int(c[o + 3]) << 24)
    return {
        "V": [int(v) for v in c[0:16]],
        "I": le16(16), "PC": le16(18), "SP": int(c[20]), "DT": int(c[21]), "ST": int(c[22]),
        "halted": int(c[23]) & 1,
        "stack": [le16(24 + 2 * k) for k in range(16)],
        "draw": le32(56), "episode": le32(60), "steps": le32(64), "prev_score": le32(68),
        "ep_ret": np.int32(np.uint32(le32(72))).item(),
        "display": c[80:336].copy(), "hist": c[336:1104].reshape(3, 256).copy(),
        "mem": c[1104:5200].copy(),
    }


def display_bits(packed256: np.ndarray) -> np.ndarray:
    """[32][64] 0/1 array from a packed 256-byte display (MSB = leftmost)."""
    return np.unpackbits(np.asarray(packed256, np.uint8).reshape(32, 8), axis=1)
