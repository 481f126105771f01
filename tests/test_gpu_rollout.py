"""Fused rollout mode (octax_rollout, SURVEY 8(d) d.3 / d.8 mode "fused", §2.3 K6 fused into
K1) vs the oracle (-m gpu).  A rollout of T steps in one launch must be bit-identical to T
single steps: every step's obs / reward / done / terminated / truncated (per-step output
buffers), the canonical states after the rollout, the episode statistics, and the ring
history that later octax_step / octax_rollout calls continue from.  Actions either come
from a caller [T][n] buffer or from the in-kernel Philox generator, which must equal the
oracle's independent implementation of the same stream (oracle.synthetic_actions)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _env(rom, spec, n, seed, offset=0):
    from paper_2510_01764_b200 import OctaxEnv
    return OctaxEnv(rom, spec, n, seed, env_offset=offset)


def _outs(T, n, per_step=True):
    shape = (T, n) if per_step else (n,)
    obs = torch.zeros(((T,) if per_step else ()) + (n, 4, 32, 8), dtype=torch.uint8, device="cuda")
    return (obs, torch.zeros(shape, dtype=torch.float32, device="cuda"),
            torch.zeros(shape, dtype=torch.uint8, device="cuda"), torch.zeros(shape, dtype=torch.uint8, device="cuda"),
            torch.zeros(shape, dtype=torch.uint8, device="cuda"))


def _check_states(g, o, ids):
    gs = g.get_states(ids)
    for k, j in enumerate(ids):
        os_ = o.get_state(j)
        if not np.array_equal(gs[k], os_):
            d = np.nonzero(gs[k] != os_)[0]
            raise AssertionError(f"env {j}: canonical state differs at bytes {d[:12]}")


def _rollout_vs_oracle(rom, spec, n, chunks, seed, aseed, offset=0, given_actions=True):
    """Consecutive rollouts of the lengths in `chunks` against the oracle stepping one step at a
    time; every step's outputs and (after each rollout) every env's canonical state compared."""
    g = _env(rom, spec, n, seed, offset)
    o = oracle.OracleEnv(rom, spec, n, seed, offset)
    na = workloads.n_actions(spec)
    t = 0
    for T in chunks:
        if given_actions:
            acts = np.stack([workloads.gen.actions(aseed, t + k, n, na) for k in range(T)])
            a_dev = torch.from_numpy(acts).cuda()
        else:
            acts = np.stack([oracle.synthetic_actions(aseed, t + k, range(offset, offset + n), na) for k in range(T)])
            a_dev = None
        obs, rew, done, term, trunc = _outs(T, n)
        g.rollout_into(T, obs, rew, done, actions=a_dev, aseed=aseed, t0=t, terminated=term, truncated=trunc)
        go, gr, gd = obs.cpu().numpy().reshape(T, n, -1), rew.cpu().numpy(), done.cpu().numpy()
        gt, gtr = term.cpu().numpy(), trunc.cpu().numpy()
        for k in range(T):
            oo, orw, od, ot, otr = o.step(acts[k])
            for name, a, b in (("obs", go[k], oo), ("reward", gr[k], orw), ("done", gd[k], od),
                               ("terminated", gt[k], ot), ("truncated", gtr[k], otr)):
                if not np.array_equal(a, b):
                    bad = np.argwhere(a != b)
                    raise AssertionError(f"rollout step {t + k}: {name} differs at {bad[:5]}")
        t += T
        _check_states(g, o, list(range(n)))
    gs, grc = g.stats()
    os_, orc = o.stats()
    assert np.array_equal(gs, os_) and grc == orc
    return g, o, gs


@pytest.mark.parametrize("game,n", [("pong_standin", 300), ("brix_standin", 257), ("target_shooter_level2", 129)])
def test_rollout_games_parity(game, n):
    rom, spec = workloads.game(game, max_episode_steps=23)
    _, _, s = _rollout_vs_oracle(rom, spec, n, [7, 1, 12, 30], 77, 5)
    assert s[1] > 0  # truncations reset envs inside the rollout


@pytest.mark.parametrize("quirks", [0, 31])
def test_rollout_fuzz_startup_quirks_parity(quirks):
    """Fuzz ROM (self-modifying stores -> dirty RAM fetches, faults, CXNN), startup segments
    (inline resets inside the rollout, no reset_kernel), all quirks."""
    rom = workloads.gen.fuzz_rom(901 + quirks, n_instr=280)
    spec = dict(workloads.DEFAULTS, score="V0 + (V1 << 8) + mem[0x300]", terminated="V2 == 9",
                action_keys=list(range(16)), quirks=quirks, max_episode_steps=17,
                startup=[(1 << 3, 2), (0, 1)])
    _, _, s = _rollout_vs_oracle(rom, spec, 200, [5, 40], 1000 + quirks, 3)
    assert s[1] > 200


@pytest.mark.parametrize("obs_format,fs", [(16, 4), (16, 2)])
def test_rollout_stack_frames_parity(obs_format, fs):
    rom, spec = workloads.game("brix_standin", obs_format=obs_format, frame_skip=fs, max_episode_steps=9)
    _rollout_vs_oracle(rom, spec, 161, [3, 14], 21, 8)


def test_rollout_generated_actions_parity():
    """actions = NULL: the in-kernel generator for steps t0..t0+T-1 (domain-1 Philox keyed by the
    GLOBAL id) equals oracle.synthetic_actions; env_offset != 0 exercises the global id."""
    rom, spec = workloads.game("pong_standin", max_episode_steps=31)
    _rollout_vs_oracle(rom, spec, 222, [9, 25, 6], workloads.ENV_SEED, workloads.ACTION_SEED,
                       offset=70000, given_actions=False)


def test_rollout_mixed_with_steps_and_overwrite_buffers():
    """Rollouts interleaved with octax_step calls (ring head continuity for T not a multiple
    of 4) and stride-0 outputs (every step overwrites one [n] buffer: the last step remains)."""
    rom, spec = workloads.game("brix_standin", max_episode_steps=13)
    n = 190
    g = _env(rom, spec, n, 3)
    o = oracle.OracleEnv(rom, spec, n, 3)
    na = workloads.n_actions(spec)
    t = 0
    for T in (3, 1, 6, 5):
        acts = np.stack([workloads.gen.actions(11, t + k, n, na) for k in range(T)])
        obs, rew, done, term, trunc = _outs(T, n, per_step=False)
        g.rollout_into(T, obs, rew, done, actions=torch.from_numpy(acts).cuda())
        for k in range(T):
            oo, orw, od, _, _ = o.step(acts[k])
        assert np.array_equal(obs.cpu().numpy().reshape(n, -1), oo)
        assert np.array_equal(rew.cpu().numpy(), orw) and np.array_equal(done.cpu().numpy(), od)
        t += T
        a1 = workloads.gen.actions(11, t, n, na)  # one plain step in between
        gobs, grew, gdone = g.step(torch.from_numpy(a1).cuda())
        oo, orw, od, _, _ = o.step(a1)
        assert np.array_equal(gobs.cpu().numpy().reshape(n, -1), oo) and np.array_equal(grew.cpu().numpy(), orw)
        t += 1
    _check_states(g, o, list(range(n)))


def test_rollout_equals_steps_on_gpu_at_4096():
    """configs[1]'s size (4,096 envs, Pong spec): a 100-step fused rollout with generated actions
    and a second handle driven by 100 octax_gen_actions + octax_step calls end in identical
    per-env state digests and identical statistics; the last obs / reward / done agree."""
    rom, spec = workloads.game("pong_standin")
    n, T = 4096, 100
    a = _env(rom, spec, n, workloads.ENV_SEED)
    b = _env(rom, spec, n, workloads.ENV_SEED)
    obs, rew, done, _, _ = _outs(T, n, per_step=False)
    a.rollout_into(T, obs, rew, done, aseed=workloads.ACTION_SEED, t0=0)
    act = torch.empty(n, dtype=torch.int32, device="cuda")
    for t in range(T):
        b.gen_actions(workloads.ACTION_SEED, t, act)
        b.step(act)
    torch.cuda.synchronize()
    assert np.array_equal(a.state_digests()[0], b.state_digests()[0])
    assert np.array_equal(a.stats()[0], b.stats()[0])
    assert torch.equal(obs, b.obs) and torch.equal(rew, b.reward) and torch.equal(done, b.done)


def test_rollout_rejects_bad_arguments():
    r = torch.zeros(64, dtype=torch.float32, device="cuda")
    d = torch.zeros(64, dtype=torch.uint8, device="cuda")
    rom, spec = workloads.game("pong_standin")
    g = _env(rom, spec, 64, 1)
    obs = torch.zeros((64, 4, 32, 8), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        g.rollout_into(4, obs, r, torch.zeros((4, 64), dtype=torch.uint8, device="cuda"))  # mixed strides


@pytest.mark.slow
def test_rollout_1M_sampled_parity_and_step_equivalence():
    """The bench's 1,048,576 envs: one 100-step fused rollout (in-kernel actions) vs the oracle on
    the config-4 sample (envs {0, 1, n/2, n-1} + 60 Philox-domain-2 ids, one oracle instance each,
    final canonical states and the last step's outputs), and vs a step-mode handle (all-env digest
    sum and statistics)."""
    rom, spec = workloads.game("pong_standin")
    n, T = 1 << 20, 100
    g = _env(rom, spec, n, workloads.ENV_SEED)
    obs, rew, done, _, _ = _outs(T, n, per_step=False)
    g.rollout_into(T, obs, rew, done, aseed=workloads.ACTION_SEED, t0=0)
    key = [workloads.ENV_SEED & 0xFFFFFFFF, workloads.ENV_SEED >> 32]
    ids = [0, 1, n // 2, n - 1] + [oracle.philox4x32_10([k, 0, 0, 2], key)[0] % n for k in range(60)]
    na = workloads.n_actions(spec)
    st = g.get_states(ids)
    go = obs.reshape(n, -1)[torch.tensor(ids, device="cuda")].cpu().numpy()
    for k, gid in enumerate(ids):
        o = oracle.OracleEnv(rom, spec, 1, workloads.ENV_SEED, gid)
        for t in range(T):
            oo, orw, od, _, _ = o.step(np.array([oracle.synthetic_action(workloads.ACTION_SEED, t, gid, na)], np.int32))
        assert np.array_equal(st[k], o.get_state(0)), gid
        assert np.array_equal(go[k], oo[0]) and rew[gid].item() == orw[0] and done[gid].item() == od[0]
    b = _env(rom, spec, n, workloads.ENV_SEED)
    act = torch.empty(n, dtype=torch.int32, device="cuda")
    for t in range(T):
        b.gen_actions(workloads.ACTION_SEED, t, act)
        b.step(act)
    assert g.state_digests()[1] == b.state_digests()[1]
    assert np.array_equal(g.stats()[0], b.stats()[0])


@pytest.mark.slow
@pytest.mark.parametrize("game", ["brix_standin", "target_shooter_level3"])
def test_rollout_config4_sampled_parity_1000_steps(game):
    """SURVEY d.1 config 4 in the fused mode: n = 262,144, ten 100-step rollouts with
    in-kernel actions; after every rollout the config-4 sample (envs {0, 1, n/2, n-1} + 60
    Philox-domain-2 ids, one oracle instance each) is compared in full canonical state, and the
    last step's obs / reward / done of the sample as well; brix's terminations reset envs inside
    the rollouts."""
    rom, spec = workloads.game(game)
    n, R, T = 262144, 10, 100
    na = workloads.n_actions(spec)
    g = _env(rom, spec, n, workloads.ENV_SEED)
    key = [workloads.ENV_SEED & 0xFFFFFFFF, workloads.ENV_SEED >> 32]
    ids = [0, 1, n // 2, n - 1] + [oracle.philox4x32_10([k, 0, 0, 2], key)[0] % n for k in range(60)]
    oracles = [oracle.OracleEnv(rom, spec, 1, workloads.ENV_SEED, gid) for gid in ids]
    idx = torch.tensor(ids, device="cuda")
    obs, rew, done, _, _ = _outs(T, n, per_step=False)
    for r in range(R):
        g.rollout_into(T, obs, rew, done, aseed=workloads.ACTION_SEED, t0=r * T)
        go = obs.reshape(n, -1)[idx].cpu().numpy()
        gr, gd = rew[idx].cpu().numpy(), done[idx].cpu().numpy()
        st = g.get_states(ids)
        for k, gid in enumerate(ids):
            for t in range(r * T, (r + 1) * T):
                oo, orw, od, _, _ = oracles[k].step(
                    np.array([oracle.synthetic_action(workloads.ACTION_SEED, t, gid, na)], np.int32))
            assert np.array_equal(st[k], oracles[k].get_state(0)), (r, gid)
            assert np.array_equal(go[k], oo[0]) and gr[k] == orw[0] and gd[k] == od[0], (r, gid)
    assert g.stats()[0][2] == n * R * T


@pytest.mark.parametrize("obs_format", [0, 16])
def test_rollout_without_obs_keeps_history(obs_format):
    """obs_out = NULL: rewards / dones (per-step strides) and states still match the oracle, and
    the display history stays intact, so the obs of a step right after the rollout is exact
    (default and stack-frames stacking)."""
    rom, spec = workloads.game("brix_standin", max_episode_steps=11, obs_format=obs_format)
    n, T = 200, 13
    g = _env(rom, spec, n, 31)
    o = oracle.OracleEnv(rom, spec, n, 31)
    na = workloads.n_actions(spec)
    acts = np.stack([workloads.gen.actions(2, k, n, na) for k in range(T)])
    _, rew, done, term, trunc = _outs(T, n)
    g.rollout_into(T, None, rew, done, actions=torch.from_numpy(acts).cuda(), terminated=term, truncated=trunc)
    for k in range(T):
        _, orw, od, ot, otr = o.step(acts[k])
        assert np.array_equal(rew[k].cpu().numpy(), orw) and np.array_equal(done[k].cpu().numpy(), od), k
        assert np.array_equal(term[k].cpu().numpy(), ot) and np.array_equal(trunc[k].cpu().numpy(), otr), k
    _check_states(g, o, list(range(n)))
    a1 = workloads.gen.actions(2, T, n, na)
    gobs, _, _ = g.step(torch.from_numpy(a1).cuda())
    oo, _, _, _, _ = o.step(a1)
    assert np.array_equal(gobs.cpu().numpy().reshape(n, -1), oo)


def test_rollout_generator_high_step_index_and_zero_length():
    """The in-kernel action generator takes the 64-bit step index t0 + t (both counter words: t0
    past 2^32) exactly like octax_gen_actions / the oracle; T = 0 is a no-op."""
    rom, spec = workloads.game("target_shooter_level1", max_episode_steps=19)
    n, T, t0 = 96, 24, (1 << 32) + 5
    g = _env(rom, spec, n, 9)
    o = oracle.OracleEnv(rom, spec, n, 9)
    obs, rew, done, _, _ = _outs(T, n)
    g.rollout_into(0, obs, rew, done, aseed=77, t0=t0)  # nothing happens
    _check_states(g, o, list(range(n)))
    g.rollout_into(T, obs, rew, done, aseed=77, t0=t0)
    na = workloads.n_actions(spec)
    for k in range(T):
        oo, orw, od, _, _ = o.step(oracle.synthetic_actions(77, t0 + k, range(n), na))
        assert np.array_equal(obs[k].cpu().numpy().reshape(n, -1), oo), k
        assert np.array_equal(rew[k].cpu().numpy(), orw) and np.array_equal(done[k].cpu().numpy(), od), k
    _check_states(g, o, list(range(n)))


@pytest.mark.slow
def test_default_horizon_truncation_10000_steps():
    """The default max_episode_steps = 10,000 (A9) at scale: 4,096 Pong-spec envs (terminated "0",
    so only truncation ends episodes) stepped 10,001 times in fused rollouts -- every env truncates
    exactly once, at step 10,000, and sampled envs match the oracle in full state afterwards."""
    rom, spec = workloads.game("pong_standin")
    assert spec["max_episode_steps"] == 10000
    n = 4096
    g = _env(rom, spec, n, workloads.ENV_SEED)
    _, rew, done, _, trunc = _outs(100, n)
    dones = 0
    for r in range(100):
        g.rollout_into(100, None, rew, done, aseed=workloads.ACTION_SEED, t0=100 * r, truncated=trunc)
        dones += int(done.sum().item())
        if r < 99:
            assert dones == 0
    assert dones == n and bool(trunc[99].all())  # all at step 10,000 (the last of rollout 99)
    _, rew1, done1, _, _ = _outs(1, n, per_step=False)
    g.rollout_into(1, None, rew1, done1, aseed=workloads.ACTION_SEED, t0=10000)
    s, _ = g.stats()
    assert s[1] == n and s[2] == n * 10001
    ids = [0, 1, 2047, n - 1]
    st = g.get_states(ids)
    na = workloads.n_actions(spec)
    for k, gid in enumerate(ids):
        o = oracle.OracleEnv(rom, spec, 1, workloads.ENV_SEED, gid)
        for t in range(10001):
            o.step(np.array([oracle.synthetic_action(workloads.ACTION_SEED, t, gid, na)], np.int32))
        assert np.array_equal(st[k], o.get_state(0)), gid


@pytest.mark.parametrize("per_step", [True, False])
def test_rollout_bool_obs_parity(per_step):
    """OCTAX_OBS_BOOL_XMAJOR handles (the paper's (4, 64, 32) boolean obs): the rollout
    kernel writes packed obs into a library staging buffer and expand_obs_kernel expands them --
    every step's with per-step strides, the last step's with stride 0 -- equal to the oracle's."""
    rom, spec = workloads.game("brix_standin", obs_format=1, max_episode_steps=7)
    n, T = 150, 9
    g = _env(rom, spec, n, 4)
    o = oracle.OracleEnv(rom, spec, n, 4)
    na = workloads.n_actions(spec)
    acts = np.stack([workloads.gen.actions(6, k, n, na) for k in range(T)])
    shape = ((T,) if per_step else ()) + (n, 4, 64, 32)
    obs = torch.zeros(shape, dtype=torch.uint8, device="cuda")
    rew = torch.zeros(((T,) if per_step else ()) + (n,), dtype=torch.float32, device="cuda")
    done = torch.zeros(((T,) if per_step else ()) + (n,), dtype=torch.uint8, device="cuda")
    g.rollout_into(T, obs, rew, done, actions=torch.from_numpy(acts).cuda())
    for k in range(T):
        oo, orw, od, _, _ = o.step(acts[k])
        if per_step:
            assert np.array_equal(obs[k].cpu().numpy().reshape(n, -1), oo), k
            assert np.array_equal(rew[k].cpu().numpy(), orw) and np.array_equal(done[k].cpu().numpy(), od), k
    if not per_step:
        assert np.array_equal(obs.cpu().numpy().reshape(n, -1), oo)
        assert np.array_equal(rew.cpu().numpy(), orw) and np.array_equal(done.cpu().numpy(), od)
    _check_states(g, o, list(range(n)))


@pytest.mark.parametrize("fseed", list(range(6)))
def test_rollout_fuzz_rom_parity(fseed):
    """The fuzz ROMs of test_gpu_parity (weighted mix of all 35 forms, self-modifying stores,
    faults, CXNN) through fused rollouts of uneven lengths, every step against the oracle."""
    rom = workloads.gen.fuzz_rom(fseed, n_instr=200 + 40 * fseed)
    spec = dict(workloads.DEFAULTS, score="V0 + (V1 << 8) + mem[0x300]", terminated="0",
                action_keys=list(range(16)), max_episode_steps=40 + 13 * fseed)
    _rollout_vs_oracle(rom, spec, 160, [11, 50, 1, 30], 1000 + fseed, fseed)
