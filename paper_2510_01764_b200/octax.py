"""Thin Python binding of the C ABI in ``include/octax.h`` (argument marshalling
only: every step of the environment runs in the CUDA kernels of liboctax.so).

torch is used for device buffers and streams only.  There is no CPU fallback:
if liboctax.so is missing or no CUDA device is present, construction raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# OCTAX_CHECKED=1 selects the bounds-checked build (device asserts; tests / debugging)
SO_PATH = os.path.join(_HERE, "liboctax_checked.so" if os.environ.get("OCTAX_CHECKED") == "1" else "liboctax.so")
# OCTAX_LIB=<path>: load another build of the same ABI (A/B timing of kernel variants)
SO_PATH = os.environ.get("OCTAX_LIB", SO_PATH)

CANON_BYTES = 5200
OBS_PACKED = 0
OBS_BOOL_XMAJOR = 1
OBS_STACK_FRAMES = 16

# every symbol include/octax.h declares
SYMBOLS = (
    "octax_create", "octax_reset", "octax_step", "octax_step_ex", "octax_step_host", "octax_step_host_frame", "octax_rollout", "octax_gen_actions",
    "octax_stats", "octax_stats_device", "octax_get_state", "octax_get_states",
    "octax_set_state", "octax_state_digests", "octax_set_kernel", "octax_get_kernel", "octax_info",
    "octax_destroy", "octax_last_error",
)
# octax_set_kernel values (include/octax.h OCTAX_KERNEL_*)
KERNELS = {"auto": 0, "lane": 1, "warp": 2}


class OctaxError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"octax status {code}: {msg}")
        self.code = code


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


class _Extras(ctypes.Structure):
    _fields_ = [("final_obs_out", ctypes.c_void_p), ("episode_return_out", ctypes.c_void_p),
                ("episode_length_out", ctypes.c_void_p), ("frame_out", ctypes.c_void_p)]


class _Opts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("cuda_stream", ctypes.c_void_p),
                ("env_offset", ctypes.c_uint64), ("total_envs", ctypes.c_uint64)]


_lib = None


def load_library():
    """Load liboctax.so (built in-tree by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        raise ImportError(f"{SO_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(SO_PATH)
    P, u64, u8p = ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint8)
    L.octax_create.argtypes = [u8p, ctypes.c_size_t, ctypes.POINTER(_Spec), u64, u64,
                               ctypes.POINTER(_Opts), ctypes.POINTER(P)]
    L.octax_reset.argtypes = [P, u64, P]
    L.octax_step.argtypes = [P, P, P, P, P, P, P]
    L.octax_step_ex.argtypes = [P, P, P, P, P, P, P, ctypes.POINTER(_Extras)]
    L.octax_step_host.argtypes = [P, P, P, P, P, P, P]
    L.octax_step_host_frame.argtypes = [P, P, P, P, P, P, P]
    L.octax_gen_actions.argtypes = [P, u64, u64, P]
    L.octax_rollout.argtypes = [P, ctypes.c_uint32, P, u64, u64, P, u64, P, P, P, P, u64]
    L.octax_stats.argtypes = [P, P]
    L.octax_stats_device.argtypes = [P, P]
    L.octax_get_state.argtypes = [P, u64, P]
    L.octax_get_states.argtypes = [P, P, u64, P]
    L.octax_set_state.argtypes = [P, u64, P]
    L.octax_state_digests.argtypes = [P, u64, u64, P, P]
    L.octax_set_kernel.argtypes = [P, ctypes.c_int]
    L.octax_get_kernel.argtypes = [P, P]
    L.octax_info.argtypes = [P, P]
    L.octax_destroy.argtypes = [P]
    L.octax_destroy.restype = None
    L.octax_last_error.restype = ctypes.c_char_p
    for name in SYMBOLS:
        if name not in ("octax_destroy", "octax_last_error"):
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc != 0:
        raise OctaxError(rc, load_library().octax_last_error().decode())


def _make_spec(spec: dict):
    keys = bytes(spec["action_keys"])
    keys_arr = (ctypes.c_uint8 * max(1, len(keys)))(*keys)
    segs = list(spec.get("startup", []))
    seg_arr = (_Seg * max(1, len(segs)))(*[_Seg(int(m), int(f)) for (m, f) in segs])
    s = _Spec()
    s.abi_version = spec.get("abi_version", 1)
    s.score_expr = None if spec.get("score") is None else spec["score"].encode()
    s.terminated_expr = None if spec.get("terminated") is None else spec["terminated"].encode()
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


def _dptr(t, dtype, n=None):
    import torch
    if t is None:
        return None
    if not (t.is_cuda and t.is_contiguous() and t.dtype == dtype):
        raise ValueError(f"expected contiguous CUDA {dtype} tensor, got {t.dtype} on {t.device}")
    if n is not None and t.numel() != n:
        raise ValueError(f"expected {n} elements, got {t.numel()}")
    return ctypes.c_void_p(t.data_ptr())


class OctaxEnv:
    """n CHIP-8 environments on one GPU: global ids env_offset .. env_offset+n-1.

    ``step(actions)`` -> (obs, reward, done) as torch CUDA tensors owned by this
    object (overwritten by the next step); ``step_into`` writes caller buffers.
    ``kernel``: "auto" (default; environment variable OCTAX_KERNEL overrides), "lane" or
    "warp" -- which step kernel runs the launches (octax_set_kernel; identical results).
    """

    def __init__(self, rom: bytes, spec: dict, n_envs: int, seed: int, device: int = 0,
                 env_offset: int = 0, total_envs: int = 0, stream=None, kernel: str | None = None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("OctaxEnv needs a CUDA device (no CPU fallback)")
        L = load_library()
        self.device = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.n = int(n_envs)
        self.spec = dict(spec)
        self.n_actions = len(spec["action_keys"]) + 1
        self.obs_format = spec.get("obs_format", OBS_PACKED) & 1
        self.obs_per_env = 1024 if self.obs_format == OBS_PACKED else 8192
        cs, self._keep = _make_spec(spec)
        rom_arr = (ctypes.c_uint8 * max(1, len(rom)))(*rom)
        opts = _Opts(device, ctypes.c_void_p(self.stream.cuda_stream), env_offset, total_envs)
        h = ctypes.c_void_p()
        _check(L.octax_create(rom_arr, len(rom), ctypes.byref(cs), self.n, seed & (2**64 - 1),
                              ctypes.byref(opts), ctypes.byref(h)))
        self._h = h
        kernel = kernel or os.environ.get("OCTAX_KERNEL", "auto")
        if kernel != "auto":
            auto = self.kernel
            self.set_kernel(kernel)
            if self.kernel != auto:  # the initial reset again, by the chosen kernel (same state)
                _check(L.octax_reset(self._h, seed & (2**64 - 1), None))
        shape = (self.n, 4, 32, 8) if self.obs_format == OBS_PACKED else (self.n, 4, 64, 32)
        self.obs = torch.zeros(shape, dtype=torch.uint8, device=self.device)
        self.reward = torch.zeros(self.n, dtype=torch.float32, device=self.device)
        self.done = torch.zeros(self.n, dtype=torch.uint8, device=self.device)
        self.terminated = torch.zeros(self.n, dtype=torch.uint8, device=self.device)
        self.truncated = torch.zeros(self.n, dtype=torch.uint8, device=self.device)

    def close(self):
        if getattr(self, "_h", None):
            load_library().octax_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reset(self, seed: int):
        _check(load_library().octax_reset(self._h, seed & (2**64 - 1), _dptr(self.obs, self.obs.dtype)))
        return self.obs

    def step_into(self, actions, obs, reward, done, terminated=None, truncated=None):
        import torch
        _check(load_library().octax_step(
            self._h, _dptr(actions, torch.int32, self.n), _dptr(obs, torch.uint8, self.n * self.obs_per_env),
            _dptr(reward, torch.float32, self.n), _dptr(done, torch.uint8, self.n),
            _dptr(terminated, torch.uint8, self.n), _dptr(truncated, torch.uint8, self.n)))

    def step(self, actions):
        self.step_into(actions, self.obs, self.reward, self.done, self.terminated, self.truncated)
        return self.obs, self.reward, self.done

    def step_ex(self, actions, final_obs=None, episode_return=None, episode_length=None):
        """Step with the optional extras of octax_step_ex (terminal obs of done envs,
        return / length of the episodes that ended this step)."""
        import torch
        ex = _Extras(None if final_obs is None else _dptr(final_obs, torch.uint8, self.n * self.obs_per_env).value,
                     None if episode_return is None else _dptr(episode_return, torch.int32, self.n).value,
                     None if episode_length is None else _dptr(episode_length, torch.int32, self.n).value)
        _check(load_library().octax_step_ex(
            self._h, _dptr(actions, torch.int32, self.n), _dptr(self.obs, torch.uint8, self.n * self.obs_per_env),
            _dptr(self.reward, torch.float32, self.n), _dptr(self.done, torch.uint8, self.n),
            _dptr(self.terminated, torch.uint8, self.n), _dptr(self.truncated, torch.uint8, self.n),
            ctypes.byref(ex)))
        return self.obs, self.reward, self.done

    def step_host(self, actions: np.ndarray, obs: np.ndarray, reward: np.ndarray, done: np.ndarray,
                  terminated: np.ndarray | None = None, truncated: np.ndarray | None = None):
        """Host-buffer step (H2D actions, D2H outputs inside the call; synchronises)."""
        p = lambda a: None if a is None else ctypes.c_void_p(a.ctypes.data)
        assert actions.dtype == np.int32 and actions.size == self.n
        _check(load_library().octax_step_host(self._h, p(actions), p(obs), p(reward), p(done),
                                              p(terminated), p(truncated)))

    def rollout_into(self, T: int, obs, reward, done, actions=None, aseed: int = 0, t0: int = 0,
                     terminated=None, truncated=None):
        """Fused rollout (octax_rollout): T steps in one launch.  actions: int32 [T, n] or None
        (in-kernel generator for steps t0..t0+T-1 under aseed).  obs: uint8 [T, n, *obs shape]
        (every step kept), [n, *obs shape] (overwritten; the last step remains) or None (no
        observations written); reward / done /
        terminated / truncated: [T, n] or [n], likewise."""
        import torch
        n, T = self.n, int(T)
        if T == 0:  # octax_rollout's no-op
            return
        ob = self.obs_per_env * n
        if obs is not None and obs.numel() not in (ob, T * ob):
            raise ValueError(f"obs must hold n or T*n observations, got {obs.numel()} bytes")
        obs_stride = ob if obs is not None and obs.numel() == T * ob and T > 1 else 0
        outs = [reward, done, terminated, truncated]
        sizes = {t.numel() for t in outs if t is not None}
        if len(sizes) != 1 or sizes.pop() not in (n, T * n):
            raise ValueError("reward / done / terminated / truncated must all be [n] or all [T, n]")
        out_stride = n if reward.numel() == T * n and T > 1 else 0
        _check(load_library().octax_rollout(
            self._h, T, _dptr(actions, torch.int32, T * n), aseed & (2**64 - 1), t0,
            _dptr(obs, torch.uint8), obs_stride, _dptr(reward, torch.float32), _dptr(done, torch.uint8),
            _dptr(terminated, torch.uint8), _dptr(truncated, torch.uint8), out_stride))

    def step_host_frame(self, actions: np.ndarray, frame: np.ndarray, reward: np.ndarray, done: np.ndarray,
                        terminated: np.ndarray | None = None, truncated: np.ndarray | None = None):
        """Host-buffer step shipping only the newest display (octax_step_host_frame): frame is
        uint8 [n, 32, 8]; the stacked obs is [d(t-3), d(t-2), d(t-1), frame], all four = frame
        where done (see include/octax.h)."""
        p = lambda a: None if a is None else ctypes.c_void_p(a.ctypes.data)
        assert actions.dtype == np.int32 and actions.size == self.n and frame.size == 256 * self.n
        _check(load_library().octax_step_host_frame(self._h, p(actions), p(frame), p(reward), p(done),
                                                    p(terminated), p(truncated)))

    def gen_actions(self, aseed: int, t: int, out):
        import torch
        _check(load_library().octax_gen_actions(self._h, aseed & (2**64 - 1), t, _dptr(out, torch.int32, self.n)))
        return out

    def stats(self):
        out = np.zeros(4, np.int64)
        rc = load_library().octax_stats(self._h, ctypes.c_void_p(out.ctypes.data))
        if rc not in (0, -8):
            _check(rc)
        return out, rc

    def stats_device(self, out):
        import torch
        _check(load_library().octax_stats_device(self._h, _dptr(out, torch.int64, 4)))
        return out

    def get_states(self, envs) -> np.ndarray:
        ids = np.ascontiguousarray(np.asarray(envs, dtype=np.uint64))
        out = np.zeros((len(ids), CANON_BYTES), np.uint8)
        _check(load_library().octax_get_states(self._h, ctypes.c_void_p(ids.ctypes.data), len(ids),
                                               ctypes.c_void_p(out.ctypes.data)))
        return out

    def get_state(self, env: int) -> np.ndarray:
        return self.get_states([env])[0]

    def set_state(self, env: int, canon: np.ndarray) -> None:
        c = np.ascontiguousarray(canon, dtype=np.uint8)
        assert c.shape == (CANON_BYTES,)
        _check(load_library().octax_set_state(self._h, env, ctypes.c_void_p(c.ctypes.data)))

    def state_digests(self, first: int = 0, count: int | None = None):
        """(digests uint64 [count], their sum mod 2^64) for local envs [first, first+count):
        FNV-1a 64 over each env's canonical state bytes (include/octax.h)."""
        n = self.n if count is None else count
        out = np.zeros(n, np.uint64)
        tot = np.zeros(1, np.uint64)
        _check(load_library().octax_state_digests(self._h, first, n, ctypes.c_void_p(out.ctypes.data),
                                                  ctypes.c_void_p(tot.ctypes.data)))
        return out, int(tot[0])

    def set_kernel(self, kernel: str) -> None:
        if kernel not in KERNELS:
            raise ValueError(f"kernel must be one of {sorted(KERNELS)}")
        _check(load_library().octax_set_kernel(self._h, KERNELS[kernel]))

    @property
    def kernel(self) -> str:
        k = ctypes.c_int(0)
        _check(load_library().octax_get_kernel(self._h, ctypes.byref(k)))
        return {1: "lane", 2: "warp"}[k.value]

    def info(self):
        out = np.zeros(4, np.uint64)
        _check(load_library().octax_info(self._h, ctypes.c_void_p(out.ctypes.data)))
        return {"n_envs": int(out[0]), "n_actions": int(out[1]), "obs_bytes": int(out[2]),
                "device_bytes": int(out[3])}
