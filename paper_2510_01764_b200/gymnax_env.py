"""Gymnax-shaped front end over OctaxEnv ("full compatibility with
both Gymnasium and Gymnax APIs").

Gymnax's functional call shapes on top of the C ABI -- argument marshalling only, every step
runs in liboctax.so:

    env = OctaxGymnaxEnv(rom, spec, num_envs=4096)
    params = env.default_params
    obs, state = env.reset(key, params)
    obs, state, reward, done, info = env.step(key, state, action, params)

Arrays carry the leading ``num_envs`` axis (Gymnax under ``jax.vmap``).  Differences from a
functional JAX env, by construction of a device-resident batch:
* the VM state lives in the library handle on the GPU; ``state`` is an :class:`EnvState` token
  (steps since reset + a generation counter).  Stepping from any state but the latest raises
  instead of branching the batch -- checkpoints go through ``OctaxEnv.get_states`` /
  ``set_state``;
* ``key`` seeds ``reset`` (an int, or a 2-word uint32 key such as ``jax.random.PRNGKey(s)``,
  words ``[hi, lo]``); ``step`` ignores it, because every random draw is counter-based and
  keyed by the reset seed, the episode and the global env id (reading A12);
* ``params`` are fixed at construction (the spec's expressions are compiled into the handle):
  passing different ones raises.
Auto-reset is same-step (reading A10, as in Gymnax): ``info["final_obs"]`` carries the terminal
observation of envs with ``done``.
"""
from __future__ import annotations

from dataclasses import dataclass

from .octax import OBS_BOOL_XMAJOR, OBS_PACKED, OctaxEnv
from .vec_env import Box, Discrete


@dataclass(frozen=True)
class EnvParams:
    max_steps_in_episode: int
    frame_skip: int
    instructions_per_frame: int
    quirks: int


@dataclass(frozen=True)
class EnvState:
    time: int        # batch steps since the last reset (per-env episode lengths: OctaxEnv.step_ex)
    generation: int  # the handle's step counter: identifies the latest state


def seed_from_key(key) -> int:
    """uint64 reset seed from an int or a 2-word uint32 key ([hi, lo], jax.random.PRNGKey layout)."""
    if isinstance(key, int):
        return key & (2**64 - 1)
    words = [int(w) & 0xFFFFFFFF for w in list(key)]
    if len(words) != 2:
        raise ValueError(f"expected an int or a 2-word uint32 key, got {len(words)} words")
    return (words[0] << 32) | words[1]


class OctaxGymnaxEnv:
    def __init__(self, rom: bytes, spec: dict, num_envs: int, device: int = 0, dense: bool = True,
                 name: str = "Octax", stream=None, kernel: str | None = None):
        fmt = OBS_BOOL_XMAJOR if dense else OBS_PACKED
        self._spec = dict(spec, obs_format=fmt)
        self.num_envs = num_envs
        self.dense = dense
        self._name = name
        self._env = OctaxEnv(rom, self._spec, num_envs, 0, device=device, stream=stream, kernel=kernel)
        self._gen = 0

    @property
    def name(self) -> str:
        return self._name

    @property
    def num_actions(self) -> int:
        return self._env.n_actions

    @property
    def default_params(self) -> EnvParams:
        s = self._spec
        return EnvParams(s.get("max_episode_steps", 10000), s.get("frame_skip", 4),
                         s.get("instructions_per_frame", 12), s.get("quirks", 0))

    def observation_space(self, params: EnvParams | None = None) -> Box:
        self._check(params)
        return Box((4, 64, 32), "bool") if self.dense else Box((4, 32, 8), "uint8", 0, 255)

    def action_space(self, params: EnvParams | None = None) -> Discrete:
        self._check(params)
        return Discrete(self._env.n_actions)

    def _check(self, params):
        if params is not None and params != self.default_params:
            raise ValueError("params are fixed at construction (compiled into the handle); "
                             f"got {params}, handle has {self.default_params}")

    def _obs(self, t):
        import torch
        v = t.view(self.num_envs, *self.observation_space().shape)
        return v.view(torch.bool) if self.dense else v

    def reset(self, key, params: EnvParams | None = None):
        self._check(params)
        obs = self._env.reset(seed_from_key(key))
        self._gen += 1
        return self._obs(obs).clone(), EnvState(0, self._gen)

    def step(self, key, state: EnvState, action, params: EnvParams | None = None):
        import torch
        self._check(params)
        if state.generation != self._gen:
            raise ValueError("stale EnvState: the batch lives on the device and only its latest state "
                             "can be stepped (checkpoint with OctaxEnv.get_states / set_state)")
        a = torch.as_tensor(action).to(device=self._env.device, dtype=torch.int32).contiguous()
        final = torch.empty(self.num_envs * self._env.obs_per_env, dtype=torch.uint8, device=self._env.device)
        obs, rew, done = self._env.step_ex(a, final_obs=final)
        self._gen += 1
        d = done.bool()
        info = {"terminated": self._env.terminated.bool(), "truncated": self._env.truncated.bool(),
                "final_obs": self._obs(final),  # valid where done
                "discount": (~d).to(torch.float32)}
        return self._obs(obs).clone(), EnvState(state.time + 1, self._gen), rew.clone(), d, info

    def close(self):
        self._env.close()
