"""Gymnasium-vector-env-shaped front end over OctaxEnv.

The paper states "full compatibility with both Gymnasium and Gymnax APIs"
(P:164).  This wrapper gives the Gymnasium vector-env call shapes on top of the
C ABI -- argument marshalling only, every step runs in liboctax.so:

    env = OctaxVecEnv(rom, spec, num_envs=4096, seed=0)
    obs, info = env.reset(seed=0)
    obs, reward, terminated, truncated, info = env.step(actions)

* auto-reset is same-step (Gymnax convention, reading A10): the returned obs of a
  finished env is its reset obs; ``info["final_obs"]`` holds the terminal obs
  (valid where ``info["_final_obs"]``), ``info["episode"]`` the finished
  episodes' return ``r`` and length ``l`` (valid where ``info["episode"]["_r"]``).
* observations are torch CUDA tensors: bool ``[n, 4, 64, 32]`` (P:146 axis order)
  when ``dense=True``, else the packed ``[n, 4, 32, 8]`` uint8 form.
* aliasing: by default (``copy=False``) ``obs`` and ``info["final_obs"]`` are
  zero-copy views of the library's persistent output buffers (the dense bool view
  reinterprets the kernel's 0/1 bytes in place, no expansion copy), valid until the
  next ``step`` / ``reset`` overwrites them -- the fast path for a learner that
  consumes the batch before stepping again.  ``copy=True`` returns clones (the
  Gymnasium habit of keeping observations across steps, e.g. in rollout buffers).
  ``reward``, ``terminated``, ``truncated`` and ``info["episode"]`` are always fresh
  tensors (n scalars each).
* ``stack="steps"`` (default, reading A3): the 4 planes are the last 4 step-end
  displays; ``stack="frames"``: the displays after the last 4 emulated frames of
  the step (OCTAX_OBS_STACK_FRAMES).
Gymnasium itself is not a dependency; ``single_observation_space`` /
``single_action_space`` are plain descriptors with ``shape`` / ``n``.
"""
from __future__ import annotations

from dataclasses import dataclass

from .octax import OBS_BOOL_XMAJOR, OBS_PACKED, OBS_STACK_FRAMES, OctaxEnv


@dataclass(frozen=True)
class Box:
    shape: tuple
    dtype: str
    low: int = 0
    high: int = 1


@dataclass(frozen=True)
class Discrete:
    n: int


class OctaxVecEnv:
    def __init__(self, rom: bytes, spec: dict, num_envs: int, seed: int = 0, device: int = 0,
                 dense: bool = True, env_offset: int = 0, stream=None, stack: str = "steps",
                 copy: bool = False, kernel: str | None = None):
        import torch
        if stack not in ("steps", "frames"):
            raise ValueError(f"stack must be 'steps' or 'frames', got {stack!r}")
        fmt = (OBS_BOOL_XMAJOR if dense else OBS_PACKED) | (OBS_STACK_FRAMES if stack == "frames" else 0)
        spec = dict(spec, obs_format=fmt)
        self._env = OctaxEnv(rom, spec, num_envs, seed, device=device, env_offset=env_offset, stream=stream,
                             kernel=kernel)
        self.num_envs = num_envs
        self.dense = dense
        self.copy = copy
        self.single_observation_space = Box((4, 64, 32), "bool") if dense else Box((4, 32, 8), "uint8", 0, 255)
        self.single_action_space = Discrete(self._env.n_actions)
        dev = self._env.device
        per = self._env.obs_per_env
        self._final = torch.zeros((num_envs, per), dtype=torch.uint8, device=dev)
        self._ret = torch.zeros(num_envs, dtype=torch.int32, device=dev)
        self._len = torch.zeros(num_envs, dtype=torch.int32, device=dev)
        self._seed = seed

    @classmethod
    def from_rom_file(cls, path: str, spec: dict, num_envs: int, **kw):
        with open(path, "rb") as f:
            return cls(f.read(), spec, num_envs, **kw)

    def _view(self, t):
        """Zero-copy: the kernel writes 0/1 bytes, reinterpreted as torch.bool in place."""
        import torch
        v = t.view(self.num_envs, *self.single_observation_space.shape)
        if self.dense:
            v = v.view(torch.bool)
        return v.clone() if self.copy else v

    def reset(self, seed: int | None = None):
        if seed is not None:
            self._seed = seed
        obs = self._env.reset(self._seed)
        return self._view(obs), {}

    def step(self, actions):
        import torch
        a = actions.to(device=self._env.device, dtype=torch.int32).contiguous()
        obs, rew, done = self._env.step_ex(a, final_obs=self._final.view(-1), episode_return=self._ret,
                                           episode_length=self._len)
        d = done.bool()
        info = {
            "final_obs": self._view(self._final), "_final_obs": d,
            "episode": {"r": self._ret.clone(), "l": self._len.clone(), "_r": d},
        }
        return self._view(obs), rew.clone(), self._env.terminated.bool(), self._env.truncated.bool(), info

    def statistics(self):
        """Integer totals since reset: {sum of returns, episodes, env steps, error flags}."""
        return self._env.stats()[0]

    def close(self):
        self._env.close()
