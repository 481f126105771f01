"""GPU <-> oracle parity (-m gpu).  The CUDA path (through the C ABI) must be
BIT-EXACT against the CPU oracle: registers, RAM, framebuffer, history,
observations, rewards, dones, episode statistics (integer work,
so the tolerance is zero; rewards are small integers stored exactly in f32)."""
from __future__ import annotations

import zlib

import numpy as np
import pytest

import oracle
import workloads
from tests.helpers import canon, hand_vectors

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _gpu_env(rom, spec, n, seed, offset=0):
    from paper_2510_01764_b200 import OctaxEnv
    return OctaxEnv(rom, spec, n, seed, env_offset=offset)


def _step_both(g, o, acts):
    a_dev = torch.from_numpy(acts).cuda()
    obs, rew, done = g.step(a_dev)
    term, trunc = g.terminated, g.truncated
    oo, orw, od, ot, otr = o.step(acts)
    return (obs.cpu().numpy().reshape(len(acts), -1), rew.cpu().numpy(), done.cpu().numpy(),
            term.cpu().numpy(), trunc.cpu().numpy()), (oo, orw, od, ot, otr)


def _assert_same(gout, oout, t):
    names = ("obs", "reward", "done", "terminated", "truncated")
    for name, a, b in zip(names, gout, oout):
        if not np.array_equal(a, b):
            bad = np.argwhere(a != b) if a.ndim > 1 else np.nonzero(a != b)[0]
            raise AssertionError(f"step {t}: {name} differs at {bad[:5]}")


def _assert_states(g, o, envs):
    gs = g.get_states(envs)
    for k, j in enumerate(envs):
        os_ = o.get_state(j)
        if not np.array_equal(gs[k], os_):
            diff = np.nonzero(gs[k] != os_)[0]
            raise AssertionError(f"env {j}: canonical state differs at bytes {diff[:12]} "
                                 f"gpu={gs[k][diff[:12]]} oracle={os_[diff[:12]]}")


def _run_parity(name_or_rom, spec, n, steps, seed, action_seed, check_every=25):
    rom = workloads.rom_bytes(name_or_rom) if isinstance(name_or_rom, str) else name_or_rom
    g = _gpu_env(rom, spec, n, seed)
    o = oracle.OracleEnv(rom, spec, n, seed)
    _assert_states(g, o, list(range(n)))
    na = len(spec["action_keys"]) + 1
    for t in range(steps):
        acts = workloads.gen.actions(action_seed, t, n, na)
        gout, oout = _step_both(g, o, acts)
        _assert_same(gout, oout, t)
        if (t + 1) % check_every == 0 or t == steps - 1:
            _assert_states(g, o, list(range(n)))
    gs, grc = g.stats()
    os_, orc = o.stats()
    assert np.array_equal(gs, os_) and grc == orc
    return g, o


# ---------------------------------------------------------------- config 1
def test_coverage_rom_n1_1000_steps_full_state_every_step():
    rom, spec = workloads.game("coverage")
    g = _gpu_env(rom, spec, 1, workloads.ENV_SEED)
    o = oracle.OracleEnv(rom, spec, 1, workloads.ENV_SEED)
    for t in range(1000):
        acts = workloads.gen.actions(1, t, 1, 17)
        gout, oout = _step_both(g, o, acts)
        _assert_same(gout, oout, t)
        _assert_states(g, o, [0])
    f = oracle.canon_fields(g.get_state(0))
    assert f["mem"][0xF00] == 20 and np.all(f["mem"][0xF01:0xF15] == 0xA5)


# ---------------------------------------------------------------- stand-in games, ragged n
@pytest.mark.parametrize("game,n", [("pong_standin", 300), ("brix_standin", 257), ("brix_standin", 1),
                                    ("target_shooter_level1", 200), ("target_shooter_level2", 333),
                                    ("target_shooter_level3", 129)])
def test_game_parity(game, n):
    rom, spec = workloads.game(game)
    _run_parity(rom, spec, n, 300, 77, 5)


@pytest.mark.parametrize("fseed", list(range(8)))
def test_fuzz_rom_parity(fseed):
    rom = workloads.gen.fuzz_rom(fseed, n_instr=200 + 40 * fseed)
    spec = dict(workloads.DEFAULTS, score="V0 + (V1 << 8) + mem[0x300]", terminated="0",
                action_keys=list(range(16)), max_episode_steps=40 + 13 * fseed)
    _run_parity(rom, spec, 160, 120, 1000 + fseed, fseed, check_every=20)


@pytest.mark.parametrize("quirks", [1, 2, 4, 8, 16, 31])
def test_quirk_parity(quirks):
    rom = workloads.gen.fuzz_rom(100 + quirks, n_instr=300)
    spec = dict(workloads.DEFAULTS, score="V5 * 3 - VF", terminated="VE == 7",
                action_keys=[1, 2, 3, 12], quirks=quirks, max_episode_steps=60)
    _run_parity(rom, spec, 130, 80, quirks, quirks)


def test_bool_obs_startup_and_truncation_parity():
    rom, spec = workloads.game("brix_standin", obs_format=1, startup=[(1 << 4, 7), (0, 3), (1 << 6, 2)],
                               max_episode_steps=33)
    _run_parity(rom, spec, 200, 100, 3, 3)


def test_frame_skip_ipf_variants_parity():
    rom, spec = workloads.game("pong_standin", frame_skip=1, instructions_per_frame=1)
    _run_parity(rom, spec, 64, 200, 9, 9)
    rom, spec = workloads.game("pong_standin", frame_skip=7, instructions_per_frame=31)
    _run_parity(rom, spec, 64, 60, 9, 9)


@pytest.mark.parametrize("quirks", [0, 31])
def test_deferred_reset_parity(quirks):
    """Specs with startup segments reset their done envs in reset_kernel, after the step
    kernel: fuzz ROMs (faults, self-modifying stores, so dirty-RAM sprite reads
    inside startup frames), short episodes so most steps reset some envs, ragged n (3 CTAs)."""
    rom = workloads.gen.fuzz_rom(77 + quirks, n_instr=240)
    spec = dict(workloads.DEFAULTS, score="V0 + mem[0x300]", terminated="V3 == 7",
                action_keys=list(range(16)), quirks=quirks, max_episode_steps=9,
                startup=[(1 << 3, 3), (0, 2)])
    g, _ = _run_parity(rom, spec, 300, 60, 5 + quirks, 6, check_every=10)
    assert g.stats()[0][1] > 300  # episodes finished: the deferred path ran


def test_reset_parity_and_obs():
    rom, spec = workloads.game("pong_standin", startup=[(2, 5)])
    g = _gpu_env(rom, spec, 50, 4)
    o = oracle.OracleEnv(rom, spec, 50, 4)
    for t in range(30):
        _step_both(g, o, workloads.gen.actions(4, t, 50, 3))
    go = g.reset(123).cpu().numpy().reshape(50, -1)
    oo = o.reset(123)
    assert np.array_equal(go, oo)
    _assert_states(g, o, list(range(50)))
    gs, _ = g.stats()
    assert list(gs) == [0, 0, 0, 0]


def test_out_of_range_actions_flag():
    rom, spec = workloads.game("pong_standin")
    g = _gpu_env(rom, spec, 40, 1)
    o = oracle.OracleEnv(rom, spec, 40, 1)
    acts = workloads.gen.actions(2, 0, 40, 3)
    acts[3], acts[17] = 9, -4
    gout, oout = _step_both(g, o, acts)
    _assert_same(gout, oout, 0)
    gs, grc = g.stats()
    os_, orc = o.stats()
    assert grc == orc == -8 and np.array_equal(gs, os_)


# ---------------------------------------------------------------- single instructions
@pytest.mark.parametrize("word,init,exp", list(hand_vectors()))
def test_hand_vector_parity(word, init, exp):
    """Each hand vector as a one-cycle step (fs=1, ipf=1) on both sides."""
    spec = dict(workloads.DEFAULTS, score="0", terminated="0", action_keys=list(range(16)),
                frame_skip=1, instructions_per_frame=1)
    rom = bytes([0x12, 0x00])
    g = _gpu_env(rom, spec, 1, 42)
    o = oracle.OracleEnv(rom, spec, 1, 42)
    f = oracle.canon_fields(o.get_state(0))
    mem = f["mem"]
    mem[0x300], mem[0x301] = word >> 8, word & 0xFF
    V = [0] * 16
    for k in range(16):
        V[k] = init.get(f"V{k:X}", init.get(f"V{k}", 0))
    stack = [init.get("STK0", 0)] + [0] * 15
    c = canon(V=V, I=init.get("I", 0), PC=0x300, SP=init.get("SP", 0), DT=init.get("DT", 0),
              ST=init.get("ST", 0), stack=stack, mem=mem, display=f["display"], hist=f["hist"])
    g.set_state(0, c)
    o.set_state(0, c)
    keys = init.get("KEYS", 0)
    action = 0 if keys == 0 else (keys & -keys).bit_length()  # key k -> action k+1
    acts = np.array([action], np.int32)
    gout, oout = _step_both(g, o, acts)
    _assert_same(gout, oout, 0)
    _assert_states(g, o, [0])


def test_set_get_state_roundtrip_random():
    rng = np.random.default_rng(5)
    rom, spec = workloads.game("pong_standin")
    g = _gpu_env(rom, spec, 3, 1)
    for _ in range(20):
        c = rng.integers(0, 256, 5200, dtype=np.uint8)
        c[20] = rng.integers(0, 17)
        c[23] &= 1
        c[76:80] = 0
        g.set_state(1, c)
        assert np.array_equal(g.get_state(1), c)


@pytest.mark.parametrize("quirks", [0, 31])
def test_random_state_fuzz_parity(quirks):
    """Arbitrary canonical states (any PC incl. odd and > 0xFFF, any stack contents, random
    RAM = every block private, random display and history) on both sides, then 6 steps:
    exercises the predecoded-table bounds, the dirty-RAM decode path and stack faults."""
    rng = np.random.default_rng(11 + quirks)
    rom, spec = workloads.game("brix_standin", quirks=quirks, max_episode_steps=0)
    n = 64
    g = _gpu_env(rom, spec, n, 9)
    o = oracle.OracleEnv(rom, spec, n, 9)
    for j in range(n):
        c = rng.integers(0, 256, 5200, dtype=np.uint8)
        c[20] = rng.integers(0, 17)
        c[23] &= 1
        c[76:80] = 0
        if j % 4 == 0:   # PC near / past the end of memory
            pc = int(rng.choice([0xFFC, 0xFFD, 0xFFE, 0xFFF, 0x1000, 0x1001, 0xFFFF]))
            c[18], c[19] = pc & 255, pc >> 8
        g.set_state(j, c)
        o.set_state(j, c)
    _assert_states(g, o, list(range(n)))
    for t in range(6):
        acts = workloads.gen.actions(12, t, n, 3)
        gout, oout = _step_both(g, o, acts)
        _assert_same(gout, oout, t)
        _assert_states(g, o, list(range(n)))


# ---------------------------------------------------------------- expressions
EXPRS = ["V5", "(V14 // 10) - (V14 % 10)", "(V9 == 0) | (V12 >= 0x3E)", "V1 == 2",
         "mem[I] + mem[I + 1] * 256", "-V3 ^ ~V4", "V1 << V2 | V3 >> V4", "V1 / V2 + V3 % V4",
         "!(V1 && V2) || V3 < V4 && V5 >= V6", "DT * ST - I", "mem[V0 * 16 + V1]",
         "((V1 + 2) * (V2 + 3) - (V3 + 4) * (V4 + 5)) / (V6 - V7 + 1)",
         "V3 // 7 - V4 % 0 + (V5 % 300) * 2 + V14 // 1 - mem[V2 // 16]"]  # fused V // c, V % c pushes


@pytest.mark.parametrize("expr", EXPRS)
def test_expression_parity(expr):
    """score: prev_score after the step must equal the oracle's parser evaluated on
    the GPU's own post-step state; terminated: GPU and oracle run the same step
    from the same random state and must agree on terminated (and everything else)."""
    rom = bytes([0x12, 0x00])
    n = 64
    rng = np.random.default_rng(zlib.crc32(expr.encode()))
    spec_s = dict(workloads.DEFAULTS, score=expr, terminated="0", action_keys=[1],
                  frame_skip=1, instructions_per_frame=1, max_episode_steps=0)
    spec_t = dict(spec_s, score="0", terminated=expr)
    gs_ = _gpu_env(rom, spec_s, n, 1)
    gt = _gpu_env(rom, spec_t, n, 1)
    ot = oracle.OracleEnv(rom, spec_t, n, 1)
    base = oracle.canon_fields(gs_.get_state(0))
    for j in range(n):
        V = rng.integers(0, 256, 16)
        V[rng.integers(0, 16)] = 0
        mem = base["mem"].copy()
        mem[0x300:0x400] = rng.integers(0, 256, 256, dtype=np.uint8)
        c = canon(V=V, I=int(rng.integers(0, 0x10000)), PC=0x200, DT=int(rng.integers(0, 256)),
                  ST=int(rng.integers(0, 256)), mem=mem, display=base["display"], hist=base["hist"])
        gs_.set_state(j, c)
        gt.set_state(j, c)
        ot.set_state(j, c)
    gs_.step(torch.zeros(n, dtype=torch.int32, device="cuda"))
    st = gs_.get_states(list(range(n)))
    for j in range(n):
        want = oracle.eval_expr(expr, st[j])
        assert oracle.canon_fields(st[j])["prev_score"] == want, j
    gout, oout = _step_both(gt, ot, np.zeros(n, np.int32))
    _assert_same(gout, oout, 0)
    _assert_states(gt, ot, list(range(n)))


# ---------------------------------------------------------------- sharding / generator
def test_shard_invariance_gpu():
    rom, spec = workloads.game("pong_standin")
    full = _gpu_env(rom, spec, 256, 8, 0)
    lo = _gpu_env(rom, spec, 128, 8, 0)
    hi = _gpu_env(rom, spec, 128, 8, 128)
    a = torch.empty(256, dtype=torch.int32, device="cuda")
    for t in range(50):
        full.gen_actions(31, t, a)
        full.step(a)
        lo.step(a[:128].contiguous())
        hi.step(a[128:].contiguous())
    s = full.get_states(list(range(256)))
    assert np.array_equal(s[:128], lo.get_states(list(range(128))))
    assert np.array_equal(s[128:], hi.get_states(list(range(128))))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_shard_invariance_r248_with_stats(world):
    """SURVEY c.3 / §8(e): R = 2, 4, 8 ragged contiguous shards (dist.shard_total) of 1,003
    global envs reproduce the single-handle run env by env (canonical state) and their
    summed int64[4] statistics equal the single handle's (the all-reduce result)."""
    from paper_2510_01764_b200 import dist
    rom, spec = workloads.game("brix_standin", max_episode_steps=40)
    total = 1003
    full = _gpu_env(rom, spec, total, 8, 0)
    parts = []
    for r in range(world):
        off, cnt = dist.shard_total(r, world, total)
        parts.append((off, cnt, _gpu_env(rom, spec, cnt, 8, off)))
    for t in range(60):
        a = torch.empty(total, dtype=torch.int32, device="cuda")
        full.gen_actions(31, t, a)
        full.step(a)
        for off, cnt, env in parts:
            b = torch.empty(cnt, dtype=torch.int32, device="cuda")
            env.gen_actions(31, t, b)            # keyed by global id: same actions
            assert torch.equal(a[off:off + cnt], b)
            env.step(b)
    s = full.get_states(list(range(total)))
    agg = np.zeros(4, np.int64)
    for off, cnt, env in parts:
        assert np.array_equal(s[off:off + cnt], env.get_states(list(range(cnt))))
        st, rc = env.stats()
        agg += st
    fs, frc = full.stats()
    assert np.array_equal(agg, fs) and fs[1] > 0
    # the per-env 64-bit state digests (SURVEY d.1 item 4) agree env by env across R
    fd, fsum = full.state_digests()
    psum = 0
    for off, cnt, env in parts:
        d, ps = env.state_digests()
        assert np.array_equal(d, fd[off:off + cnt])
        psum = (psum + ps) % 2**64
    assert psum == fsum


def _fnv1a64(b: bytes) -> int:
    h = 0xCBF29CE484222325
    for x in b:
        h = ((h ^ x) * 0x100000001B3) % 2**64
    return h


def test_state_digests_definition():
    """octax_state_digests = FNV-1a 64 of the canonical bytes (include/octax.h), written out
    here independently, on sampled envs of a ragged handle after divergent steps; sub-ranges
    and chunking (count > 65,536) agree with the full range; bad ranges are refused."""
    rom, spec = workloads.game("brix_standin", max_episode_steps=30)
    n = 70_001
    g = _gpu_env(rom, spec, n, 3)
    a = torch.empty(n, dtype=torch.int32, device="cuda")
    for t in range(12):
        g.gen_actions(5, t, a)
        g.step(a)
    d, tot = g.state_digests()
    assert tot == int(d.astype(object).sum()) % 2**64
    ids = [0, 1, 127, 128, 65535, 65536, n - 1]
    canon = g.get_states(ids)
    for j, c in zip(ids, canon):
        assert int(d[j]) == _fnv1a64(bytes(c))
    d2, _ = g.state_digests(65530, 20)
    assert np.array_equal(d2, d[65530:65550])
    assert len(np.unique(d)) > n // 2   # distinct states hash apart
    from paper_2510_01764_b200.octax import OctaxError
    with pytest.raises(OctaxError):
        g.state_digests(n - 5, 10)


def test_gen_actions_matches_oracle_generator():
    rom, spec = workloads.game("coverage")
    g = _gpu_env(rom, spec, 1000, 1, 5000)
    a = torch.empty(1000, dtype=torch.int32, device="cuda")
    for t in (0, 1, 2**32 + 7):
        g.gen_actions(0xABCDEF0123, t, a)
        want = oracle.synthetic_actions(0xABCDEF0123, t, range(5000, 6000), 17)
        assert np.array_equal(a.cpu().numpy(), want)


# ---------------------------------------------------------------- full size, bench launch config
@pytest.mark.slow
def test_full_size_sampled_parity():
    """n = 1,048,576 (bench workload), device-generated actions, 64 sampled envs
    re-simulated one by one by the oracle (SURVEY d.1 config 4 sampling)."""
    rom, spec = workloads.game("pong_standin")
    n, T = 1 << 20, 40
    g = _gpu_env(rom, spec, n, workloads.ENV_SEED)
    a = torch.empty(n, dtype=torch.int32, device="cuda")
    key = [workloads.ENV_SEED & 0xFFFFFFFF, workloads.ENV_SEED >> 32]
    ids = [0, 1, n // 2, n - 1] + [oracle.philox4x32_10([k, 0, 0, 2], key)[0] % n for k in range(60)]
    oracles = [oracle.OracleEnv(rom, spec, 1, workloads.ENV_SEED, gid) for gid in ids]
    idx = torch.tensor(ids, device="cuda")
    for t in range(T):
        g.gen_actions(workloads.ACTION_SEED, t, a)
        obs, rew, done = g.step(a)
        go = obs.reshape(n, -1)[idx].cpu().numpy()
        gr = rew[idx].cpu().numpy()
        gd = done[idx].cpu().numpy()
        for k, gid in enumerate(ids):
            act = np.array([oracle.synthetic_action(workloads.ACTION_SEED, t, gid, 3)], np.int32)
            oo, orw, od, _, _ = oracles[k].step(act)
            assert np.array_equal(go[k], oo[0]) and gr[k] == orw[0] and gd[k] == od[0], (t, gid)
    st = g.get_states(ids)
    for k in range(len(ids)):
        assert np.array_equal(st[k], oracles[k].get_state(0))
    s, _ = g.stats()
    assert s[2] == n * T


@pytest.mark.slow
@pytest.mark.parametrize("game", ["pong_standin", "brix_standin", "target_shooter_level1",
                                  "target_shooter_level2", "target_shooter_level3"])
def test_config4_sampled_parity_1000_steps(game):
    """SURVEY d.1 config 4 as specified: n = 262,144, T = 1,000 steps with device-generated
    random actions; envs {0, 1, n/2, n-1} + 60 Philox-domain-2 ids gathered on device every
    step and compared with one oracle instance each; final canonical states compared."""
    rom, spec = workloads.game(game)
    n, T = 262144, 1000
    na = workloads.n_actions(spec)
    g = _gpu_env(rom, spec, n, workloads.ENV_SEED)
    a = torch.empty(n, dtype=torch.int32, device="cuda")
    key = [workloads.ENV_SEED & 0xFFFFFFFF, workloads.ENV_SEED >> 32]
    ids = [0, 1, n // 2, n - 1] + [oracle.philox4x32_10([k, 0, 0, 2], key)[0] % n for k in range(60)]
    oracles = [oracle.OracleEnv(rom, spec, 1, workloads.ENV_SEED, gid) for gid in ids]
    idx = torch.tensor(ids, device="cuda")
    for t in range(T):
        g.gen_actions(workloads.ACTION_SEED, t, a)
        obs, rew, done = g.step(a)
        go = obs.reshape(n, -1)[idx].cpu().numpy()
        gr = rew[idx].cpu().numpy()
        gd = done[idx].cpu().numpy()
        for k, gid in enumerate(ids):
            act = np.array([oracle.synthetic_action(workloads.ACTION_SEED, t, gid, na)], np.int32)
            oo, orw, od, _, _ = oracles[k].step(act)
            assert np.array_equal(go[k], oo[0]) and gr[k] == orw[0] and gd[k] == od[0], (t, gid)
    st = g.get_states(ids)
    for k in range(len(ids)):
        assert np.array_equal(st[k], oracles[k].get_state(0)), ids[k]


def test_cuda_graph_capture_matches_eager():
    """Steps captured in a CUDA graph (bench sweep mode) give the same states as eager launches."""
    from paper_2510_01764_b200 import OctaxEnv
    rom, spec = workloads.game("brix_standin")
    n, K = 700, 8
    s = torch.cuda.Stream()
    eager = OctaxEnv(rom, spec, n, 5)
    graphed = OctaxEnv(rom, spec, n, 5, stream=s)
    acts = torch.empty((2 * K, n), dtype=torch.int32, device="cuda")
    for t in range(2 * K):
        eager.gen_actions(77, t, acts[t])
    torch.cuda.synchronize()
    for t in range(2 * K):
        eager.step(acts[t])
    g = torch.cuda.CUDAGraph()
    obs, rew, done = graphed.obs, graphed.reward, graphed.done
    with torch.cuda.graph(g, stream=s):
        for k in range(K):
            graphed.step_into(acts[k], obs, rew, done)
    # the capture itself runs nothing: replay twice = 2K steps, but actions repeat -> compare
    # against an eager run with the same repeated action schedule
    ref = OctaxEnv(rom, spec, n, 5)
    for rep in range(2):
        with torch.cuda.stream(s):
            g.replay()
        for k in range(K):
            ref.step(acts[k])
    torch.cuda.synchronize()
    ids = list(range(0, n, 7))
    assert np.array_equal(graphed.get_states(ids), ref.get_states(ids))
    assert np.array_equal(graphed.obs.cpu().numpy(), ref.obs.cpu().numpy())


@pytest.mark.parametrize("obs_format", [0, 1])
def test_step_ex_final_obs_and_episode_info(obs_format):
    """octax_step_ex extras vs the oracle: terminal obs of done envs (SPEC S:409
    convention), return and length of the finished episodes."""
    rom, spec = workloads.game("brix_standin", obs_format=obs_format, max_episode_steps=45)
    n = 300
    g = _gpu_env(rom, spec, n, 21)
    o = oracle.OracleEnv(rom, spec, n, 21)
    per = g.obs_per_env
    fin = torch.zeros(n * per, dtype=torch.uint8, device="cuda")
    er = torch.zeros(n, dtype=torch.int32, device="cuda")
    el = torch.zeros(n, dtype=torch.int32, device="cuda")
    seen = 0
    for t in range(120):
        acts = workloads.gen.actions(21, t, n, 3)
        g.step_ex(torch.from_numpy(acts).cuda(), final_obs=fin, episode_return=er, episode_length=el)
        oo, orw, od, ot, otr, ofin, oer, oel = o.step_ex(acts)
        assert np.array_equal(g.obs.cpu().numpy().reshape(n, -1), oo)
        assert np.array_equal(g.done.cpu().numpy(), od)
        assert np.array_equal(er.cpu().numpy(), oer)
        assert np.array_equal(el.cpu().numpy().astype(np.uint32), oel)
        d = od.astype(bool)
        if d.any():
            gf = fin.cpu().numpy().reshape(n, -1)
            assert np.array_equal(gf[d], ofin[d])
            seen += int(d.sum())
    assert seen > 20


@pytest.mark.parametrize("obs_format,fs", [(16, 4), (16, 1), (16, 2), (16, 6), (17, 4), (17, 3)])
def test_stack_frames_obs_parity(obs_format, fs):
    """OCTAX_OBS_STACK_FRAMES: obs = the displays after the last 4 frames of the step
    (per-frame smem->HBM stores inside the kernel), incl. terminal final_obs and
    same-step resets, bit-exact vs the oracle."""
    rom, spec = workloads.game("brix_standin", obs_format=obs_format, frame_skip=fs, max_episode_steps=33)
    n = 291
    g = _gpu_env(rom, spec, n, 17)
    o = oracle.OracleEnv(rom, spec, n, 17)
    fin = torch.zeros(n * g.obs_per_env, dtype=torch.uint8, device="cuda")
    seen = 0
    for t in range(80):
        acts = workloads.gen.actions(5, t, n, 3)
        g.step_ex(torch.from_numpy(acts).cuda(), final_obs=fin)
        oo, orw, od, ot, otr, ofin, oer, oel = o.step_ex(acts)
        assert np.array_equal(g.obs.cpu().numpy().reshape(n, -1), oo), t
        assert np.array_equal(g.reward.cpu().numpy(), orw), t
        d = od.astype(bool)
        if d.any():
            assert np.array_equal(fin.cpu().numpy().reshape(n, -1)[d], ofin[d]), t
            seen += int(d.sum())
    _assert_states(g, o, list(range(0, n, 7)))
    assert seen > 0


def test_vec_env_wrapper_shapes_and_values():
    from paper_2510_01764_b200.vec_env import OctaxVecEnv
    rom, spec = workloads.game("brix_standin", max_episode_steps=30)
    n = 64
    env = OctaxVecEnv(rom, spec, n, seed=3, dense=True)
    o = oracle.OracleEnv(rom, dict(spec, obs_format=1), n, 3)
    obs, info = env.reset(seed=3)
    assert obs.shape == (n, 4, 64, 32) and obs.dtype == torch.bool
    assert np.array_equal(obs.cpu().numpy().reshape(n, -1).astype(np.uint8), o.reset(3))
    for t in range(40):
        acts = workloads.gen.actions(8, t, n, env.single_action_space.n)
        obs, rew, term, trunc, info = env.step(torch.from_numpy(acts))
        oo, orw, od, ot, otr, ofin, oer, oel = o.step_ex(acts)
        assert np.array_equal(obs.cpu().numpy().reshape(n, -1).astype(np.uint8), oo)
        assert np.array_equal(rew.cpu().numpy(), orw)
        assert np.array_equal(term.cpu().numpy(), ot.astype(bool))
        assert np.array_equal(trunc.cpu().numpy(), otr.astype(bool))
        m = info["_final_obs"].cpu().numpy()
        assert np.array_equal(m, od.astype(bool))
        if m.any():
            fo = info["final_obs"].cpu().numpy().reshape(n, -1).astype(np.uint8)
            assert np.array_equal(fo[m], ofin[m])
            assert np.array_equal(info["episode"]["r"].cpu().numpy()[m], oer[m])


EDGE_CASES = [(name, 0) for name in __import__("workloads.edge_roms", fromlist=["EDGE_ROMS"]).EDGE_ROMS] + \
             [("draw_edges", 8), ("flags", 1 | 16), ("self_modify", 2)]


@pytest.mark.parametrize("name,quirks", EDGE_CASES)
def test_edge_rom_parity(name, quirks):
    """SURVEY c.7 edge-case ROMs (self-modifying code, odd / boundary PCs, address
    wrap, draw clipping / wrap / DXY0, X=Y=F flags, deep calls, key waits, timers,
    RNG across resets), ragged n, bit-exact including full canonical state."""
    from workloads import edge_roms
    src, over = edge_roms.EDGE_ROMS[name]
    spec = dict(workloads.DEFAULTS, score="V6 + (V1 << 8) + mem[0x300]", terminated="0",
                action_keys=list(range(16)), max_episode_steps=150, quirks=quirks)
    spec.update(over)
    _run_parity(edge_roms.rom(name), spec, 97, 160, 11 + quirks, 7, check_every=16)


@pytest.mark.slow
@pytest.mark.parametrize("quirks", [0, 31])
def test_decode_totality_gpu(quirks):
    """SURVEY c.5: every one of the 65,536 instruction words executed once on the GPU, one
    env per word, from random register / stack / timer state (PC = 0x300, one cycle per
    step): halts exactly where the oracle halts and on no valid word, and the full
    canonical state after the cycle matches the oracle for every env."""
    from tests.test_oracle_pins import _valid_word
    rng = np.random.default_rng(65536 + quirks)
    rom, spec = workloads.game("brix_standin", quirks=quirks, frame_skip=1, instructions_per_frame=1,
                               max_episode_steps=0, terminated="0", score="V0 + VF * 256 + I")
    n = 65536
    g = _gpu_env(rom, spec, n, 3)
    o = oracle.OracleEnv(rom, spec, n, 3)
    base = g.get_state(0)
    sp = rng.integers(0, 17, n)
    for w in range(n):
        c = base.copy()
        c[0:16] = rng.integers(0, 256, 16)
        I = int(rng.integers(0, 0x1000))
        c[16], c[17] = I & 255, I >> 8
        c[18], c[19] = 0x00, 0x03                     # PC = 0x300
        c[20] = sp[w]
        c[21], c[22] = rng.integers(0, 256, 2)
        c[24:56] = rng.integers(0, 256, 32)           # arbitrary return addresses
        c[1104 + 0x300], c[1104 + 0x301] = w >> 8, w & 255
        g.set_state(w, c)
        o.set_state(w, c)
    acts = workloads.gen.actions(17, 0, n, 3)
    gout, oout = _step_both(g, o, acts)
    _assert_same(gout, oout, 0)
    done = oout[2].astype(bool)
    ok_sp = (sp >= 1) & (sp <= 15)
    valid = np.array([_valid_word(w) for w in range(n)])
    assert not (done & valid & ok_sp).any()           # valid words never fault with a safe SP
    assert done[~valid].all()                         # invalid words always halt
    for lo in range(0, n, 4096):
        ids = list(range(lo, lo + 4096))
        gs = g.get_states(ids)
        for j in ids:
            if not np.array_equal(gs[j - lo], o.get_state(j)):
                raise AssertionError(f"state differs for word {j:04X}")


def test_font_bytes_golden_gpu():
    """The CUDA path's power-on image holds SURVEY App. B's 80 font bytes (tests/golden/font.txt)
    -- its table is a transcription independent of the oracle's, so both are pinned to the golden."""
    from tests.helpers import golden_lines
    font = bytes(int(b, 16) for line in golden_lines("font.txt") for b in line.split()[1:])
    rom, spec = workloads.game("pong_standin")
    g = _gpu_env(rom, spec, 3, 1)
    for c in g.get_states([0, 2]):
        assert bytes(oracle.canon_fields(c)["mem"][0x50:0xA0]) == font


@pytest.mark.parametrize("dense", [True, False])
def test_vec_env_zero_copy_and_copy_mode(dense):
    """OctaxVecEnv's default obs is a zero-copy view of the library's output buffer (the bool
    view reinterprets the kernel's 0/1 bytes: same data_ptr, no 8 KB/env expansion copy);
    copy=True returns clones that survive the next step (Gymnasium rollout-buffer habit)."""
    from paper_2510_01764_b200.vec_env import OctaxVecEnv
    rom, spec = workloads.game("brix_standin", max_episode_steps=30)
    n = 96
    fast = OctaxVecEnv(rom, spec, n, seed=3, dense=dense)
    safe = OctaxVecEnv(rom, spec, n, seed=3, dense=dense, copy=True)
    obs, _ = fast.reset(seed=3)
    assert obs.data_ptr() == fast._env.obs.data_ptr()
    assert obs.dtype == (torch.bool if dense else torch.uint8)
    sobs, _ = safe.reset(seed=3)
    assert sobs.data_ptr() != safe._env.obs.data_ptr() and torch.equal(obs, sobs)
    kept = []
    for t in range(12):
        a = torch.from_numpy(workloads.gen.actions(8, t, n, fast.single_action_space.n))
        o1, r1, te1, tr1, i1 = fast.step(a)
        o2, r2, te2, tr2, i2 = safe.step(a)
        assert o1.data_ptr() == fast._env.obs.data_ptr()
        assert i1["final_obs"].data_ptr() == fast._final.data_ptr()
        assert torch.equal(o1, o2) and torch.equal(r1, r2) and torch.equal(te1, te2)
        kept.append((o2, o1.clone(), i2["episode"]["r"], i1["episode"]["r"].clone()))
    for o2, o1c, r2, r1c in kept:   # copies kept across steps are still the step's values
        assert torch.equal(o2, o1c) and torch.equal(r2, r1c)


# ---------------------------------------------------------------- full-size sampled parity helper
def _sampled_parity(rom, spec, n, T, extra_ids=(), check_every=None):
    """n envs on the GPU with device-generated actions; the SURVEY d.1 config-4 sample
    ({0, 1, n/2, n-1} + 60 Philox domain-2 ids + extra_ids) re-simulated one oracle instance
    each; obs / reward / done gathered on device every step, final canonical states compared
    (and every `check_every` steps)."""
    na = workloads.n_actions(spec)
    g = _gpu_env(rom, spec, n, workloads.ENV_SEED)
    a = torch.empty(n, dtype=torch.int32, device="cuda")
    key = [workloads.ENV_SEED & 0xFFFFFFFF, workloads.ENV_SEED >> 32]
    ids = [0, 1, n // 2, n - 1] + [oracle.philox4x32_10([k, 0, 0, 2], key)[0] % n for k in range(60)]
    ids += [i for i in extra_ids if i < n]
    oracles = [oracle.OracleEnv(rom, spec, 1, workloads.ENV_SEED, gid) for gid in ids]
    idx = torch.tensor(ids, device="cuda")
    dones = 0
    for t in range(T):
        g.gen_actions(workloads.ACTION_SEED, t, a)
        obs, rew, done = g.step(a)
        go = obs.reshape(n, -1)[idx].cpu().numpy()
        gr = rew[idx].cpu().numpy()
        gd = done[idx].cpu().numpy()
        dones += int(done.sum().item())
        for k, gid in enumerate(ids):
            act = np.array([oracle.synthetic_action(workloads.ACTION_SEED, t, gid, na)], np.int32)
            oo, orw, od, _, _ = oracles[k].step(act)
            assert np.array_equal(go[k], oo[0]) and gr[k] == orw[0] and gd[k] == od[0], (t, gid)
        if check_every and (t + 1) % check_every == 0:
            st = g.get_states(ids)
            for k in range(len(ids)):
                assert np.array_equal(st[k], oracles[k].get_state(0)), (t, ids[k])
    st = g.get_states(ids)
    for k in range(len(ids)):
        assert np.array_equal(st[k], oracles[k].get_state(0)), ids[k]
    s, rc = g.stats()
    assert s[2] == n * T
    return g, dones


@pytest.mark.slow
@pytest.mark.parametrize("game", ["pong_standin", "brix_standin"])
def test_reset_kernel_multipass_sampled_parity(game):
    """Deferred resets (specs with startup segments) when one step resets far more envs than
    reset_kernel's grid holds (148 SMs x 5 CTAs x 128 = 94,720): all 262,144 envs were created
    together and truncate on the same steps (max_episode_steps = 5), so steps 5 and 10 reset
    every env in one launch -- 3 grid-stride passes reusing the CTA's shared-memory slots
    (VERDICT r1 weak #2).  The config-4 sample plus ids around the pass-size
    boundaries are compared step by step, full canonical state every 5 steps."""
    rom, spec = workloads.game(game, startup=[(0, 3), (1 << 1, 2)], max_episode_steps=5)
    n = 262144
    passes = [94720 * k + j for k in range(3) for j in (0, 127, 128, 94719) if 94720 * k + j < n]
    g, dones = _sampled_parity(rom, spec, n, 12, extra_ids=passes, check_every=5)
    assert dones >= 2 * n  # the synchronized truncations happened
    s, _ = g.stats()
    assert s[1] >= 2 * n


@pytest.mark.slow
def test_bool_obs_1M_sampled_parity():
    """OCTAX_OBS_BOOL_XMAJOR at the bench's 1,048,576 envs (the 8 KB/env expand_obs_kernel
    path the bool-obs throughput is quoted on), 64 sampled envs vs the oracle's bool obs."""
    rom, spec = workloads.game("pong_standin", obs_format=1)
    _sampled_parity(rom, spec, 1 << 20, 24)


@pytest.mark.slow
def test_stack_frames_1M_sampled_parity():
    """OCTAX_OBS_STACK_FRAMES (per-frame obs planes written inside the step kernel) at
    1,048,576 envs, with truncation so same-step resets occur in the sample."""
    rom, spec = workloads.game("brix_standin", obs_format=16, max_episode_steps=11)
    _sampled_parity(rom, spec, 1 << 20, 24)


@pytest.mark.parametrize("obs_format,quirks", [(16, 31), (17, 31), (16, 0)])
def test_stack_frames_startup_quirks_parity(obs_format, quirks):
    """OCTAX_OBS_STACK_FRAMES x startup segments (deferred resets writing the reset display to
    all planes) x all quirks, ragged n, full state: the combination VERDICT r1 found untested."""
    rom = workloads.gen.fuzz_rom(501 + quirks, n_instr=260)
    spec = dict(workloads.DEFAULTS, score="V0 + mem[0x300]", terminated="V3 == 7",
                action_keys=list(range(16)), quirks=quirks, max_episode_steps=13,
                startup=[(1 << 5, 2), (0, 3)], obs_format=obs_format, frame_skip=3)
    g, _ = _run_parity(rom, spec, 333, 60, 41 + quirks, 4, check_every=10)
    assert g.stats()[0][1] > 333


@pytest.mark.parametrize("game,n,startup", [("brix_standin", 333, None), ("pong_standin", 130, [(1 << 1, 3)])])
def test_step_host_frame_reconstructs_obs(game, n, startup):
    """octax_step_host_frame ships only the newest display; a host history started from the reset
    obs and rebuilt as [d(t-3), d(t-2), d(t-1), frame] (all four = frame where done, A10) equals
    the oracle's stacked obs at every step, and reward / done / terminated / truncated match."""
    over = dict(max_episode_steps=9)
    if startup:
        over["startup"] = startup
    rom, spec = workloads.game(game, **over)
    g = _gpu_env(rom, spec, n, 17)
    o = oracle.OracleEnv(rom, spec, n, 17)
    hist = g.reset(17).cpu().numpy().reshape(n, 4, 256)[:, 1:].copy()  # d(t-3), d(t-2), d(t-1)
    o.reset(17)
    na = workloads.n_actions(spec)
    frame = np.zeros((n, 32, 8), np.uint8)
    rew, done = np.zeros(n, np.float32), np.zeros(n, np.uint8)
    term, trunc = np.zeros(n, np.uint8), np.zeros(n, np.uint8)
    for t in range(40):
        acts = np.ascontiguousarray(workloads.gen.actions(23, t, n, na))
        g.step_host_frame(acts, frame, rew, done, term, trunc)
        f = frame.reshape(n, 256)
        obs = np.concatenate([hist, f[:, None]], axis=1)
        obs[done != 0] = f[done != 0][:, None]
        oo, orw, od, ot, otr = o.step(acts)
        assert np.array_equal(obs.reshape(n, -1), oo), t
        assert np.array_equal(rew, orw) and np.array_equal(done, od), t
        assert np.array_equal(term, ot) and np.array_equal(trunc, otr), t
        hist = obs[:, 1:].copy()
    assert o.stats()[0][1] > 0  # truncations / resets happened


def test_gymnax_env_matches_oracle():
    """OctaxGymnaxEnv (Gymnax call shapes, NEXT-3): reset(key) seeds like octax_reset(seed),
    step(key, state, action) returns the oracle's obs / reward / done (bool x-major obs),
    terminal obs in info where done; a stale EnvState is refused."""
    from paper_2510_01764_b200.gymnax_env import OctaxGymnaxEnv, seed_from_key
    rom, spec = workloads.game("brix_standin", max_episode_steps=6)
    n = 100
    env = OctaxGymnaxEnv(rom, spec, n)
    key = [0x12345678, 0x9ABCDEF0]
    o = oracle.OracleEnv(rom, dict(spec, obs_format=1), n, seed_from_key(key))
    obs, state = env.reset(key, env.default_params)
    assert np.array_equal(obs.cpu().numpy().reshape(n, -1).astype(np.uint8), o.reset(seed_from_key(key)))
    na = env.num_actions
    for t in range(10):
        a = workloads.gen.actions(5, t, n, na)
        old = state
        obs, state, rew, done, info = env.step(None, state, torch.from_numpy(a))
        oo, orw, od, ot, otr = o.step(a)
        assert np.array_equal(obs.cpu().numpy().reshape(n, -1).astype(np.uint8), oo), t
        assert np.array_equal(rew.cpu().numpy(), orw) and np.array_equal(done.cpu().numpy().astype(np.uint8), od)
        assert np.array_equal(info["truncated"].cpu().numpy().astype(np.uint8), otr)
    assert state.time == 10
    with pytest.raises(ValueError):
        env.step(None, old, torch.from_numpy(a))
    env.close()


@pytest.mark.slow
@pytest.mark.parametrize("startup,obs_format", [(None, 0), ([(1 << 1, 2)], 0), (None, 1)])
def test_pipelined_host_steps_match_device_steps(startup, obs_format):
    """octax_step_host / octax_step_host_frame at 262,144 envs step the envs in several chunk
    launches whose device->host copies overlap the next chunk's kernel: outputs equal a twin
    handle stepped with octax_step on the device, step by step, including synchronized
    truncations (deferred resets per chunk when the spec has startup segments)."""
    from paper_2510_01764_b200 import OctaxEnv
    over = dict(max_episode_steps=3)
    if startup:
        over["startup"] = startup
    rom, spec = workloads.game("brix_standin", obs_format=obs_format, **over)
    n = 262144
    host_full, host_frame, dev = (OctaxEnv(rom, spec, n, 5) for _ in range(3))
    na = workloads.n_actions(spec)
    per = host_full.obs_per_env
    o_h = np.zeros((n, per), np.uint8)
    f_h = np.zeros((n, 32, 8), np.uint8)
    r1, r2 = np.zeros(n, np.float32), np.zeros(n, np.float32)
    d1, d2 = np.zeros(n, np.uint8), np.zeros(n, np.uint8)
    t1, t2 = np.zeros(n, np.uint8), np.zeros(n, np.uint8)
    for t in range(7):
        a = np.ascontiguousarray(workloads.gen.actions(3, t, n, na))
        host_full.step_host(a, o_h, r1, d1, t1)
        host_frame.step_host_frame(a, f_h, r2, d2, t2)
        obs, rew, done = dev.step(torch.from_numpy(a).cuda())
        ob = obs.cpu().numpy().reshape(n, per)
        assert np.array_equal(o_h, ob), t
        if obs_format == 0:  # the frame is obs plane 3 in the packed layout
            assert np.array_equal(f_h.reshape(n, 256), ob[:, 768:]), t
        else:                # bool x-major plane 3 = the frame's pixels, transposed
            bits = np.unpackbits(f_h.reshape(n, 32, 8), axis=2)          # [n][y][x]
            assert np.array_equal(bits.transpose(0, 2, 1).reshape(n, 2048), ob[:, 3 * 2048:]), t
        rw, dn, tm = rew.cpu().numpy(), done.cpu().numpy(), dev.terminated.cpu().numpy()
        for r_, d_, t_ in ((r1, d1, t1), (r2, d2, t2)):
            assert np.array_equal(r_, rw) and np.array_equal(d_, dn) and np.array_equal(t_, tm), t
    assert d1.sum() > 0 or dev.stats()[0][1] > 0
    for e in (host_full, host_frame, dev):
        assert np.array_equal(e.state_digests()[0][:4096], dev.state_digests()[0][:4096])


@pytest.mark.slow
def test_max_size_16M_envs_sampled_parity():
    """Maximum sizes: 16,777,293 envs (2^24 + 77, a ragged last CTA) on one B200 -- ~87 GB of VM
    state plus 17 GB of packed obs, byte offsets far past 2^32 in every per-env array.  Three steps
    (one of them a fused rollout of two steps) with device-generated actions; envs near the ends of
    the range and around 2^24 are compared with the oracle in full canonical state and outputs."""
    rom, spec = workloads.game("brix_standin", max_episode_steps=2)
    n = (1 << 24) + 77
    g = _gpu_env(rom, spec, n, workloads.ENV_SEED)
    ids = [0, 1, 127, 128, (1 << 23) + 5, (1 << 24) - 1, 1 << 24, n - 2, n - 1]
    oracles = [oracle.OracleEnv(rom, spec, 1, workloads.ENV_SEED, gid) for gid in ids]
    na = workloads.n_actions(spec)
    a = torch.empty(n, dtype=torch.int32, device="cuda")
    idx = torch.tensor(ids, device="cuda")
    g.gen_actions(workloads.ACTION_SEED, 0, a)
    obs, rew, done = g.step(a)
    go, gr, gd = obs.reshape(n, -1)[idx].cpu().numpy(), rew[idx].cpu().numpy(), done[idx].cpu().numpy()
    for k, gid in enumerate(ids):
        oo, orw, od, _, _ = oracles[k].step(np.array([oracle.synthetic_action(workloads.ACTION_SEED, 0, gid, na)], np.int32))
        assert np.array_equal(go[k], oo[0]) and gr[k] == orw[0] and gd[k] == od[0], gid
    g.rollout_into(2, g.obs, g.reward, g.done, aseed=workloads.ACTION_SEED, t0=1)
    go, gr, gd = g.obs.reshape(n, -1)[idx].cpu().numpy(), g.reward[idx].cpu().numpy(), g.done[idx].cpu().numpy()
    st = g.get_states(ids)
    for k, gid in enumerate(ids):
        for t in (1, 2):
            oo, orw, od, _, _ = oracles[k].step(np.array([oracle.synthetic_action(workloads.ACTION_SEED, t, gid, na)], np.int32))
        assert np.array_equal(go[k], oo[0]) and gr[k] == orw[0] and gd[k] == od[0], gid
        assert np.array_equal(st[k], oracles[k].get_state(0)), gid
    s, _ = g.stats()
    assert s[2] == 3 * n and s[1] >= n  # every env truncated at step 2 (max_episode_steps = 2)
    g.close()


def test_concurrent_handles_on_separate_streams():
    """Handles are independent (include/octax.h): three games, each on its own CUDA stream,
    launched interleaved without synchronisation between them, match
    their oracles; a fourth handle on the default stream shares the device meanwhile."""
    from paper_2510_01764_b200 import OctaxEnv
    games = [("pong_standin", 300), ("brix_standin", 257), ("target_shooter_level1", 129)]
    streams = [torch.cuda.Stream() for _ in games]
    envs, oracles, specs = [], [], []
    for (game, n), s in zip(games, streams):
        rom, spec = workloads.game(game, max_episode_steps=9)
        envs.append(OctaxEnv(rom, spec, n, 11, stream=s))
        oracles.append(oracle.OracleEnv(rom, spec, n, 11))
        specs.append(spec)
    rom, spec = workloads.game("coverage")
    bystander = OctaxEnv(rom, spec, 4096, 3)
    acts = [[torch.from_numpy(workloads.gen.actions(7, t, n, workloads.n_actions(sp))).cuda()
             for t in range(12)] for (g, n), sp in zip(games, specs)]
    outs = [[] for _ in games]
    torch.cuda.synchronize()
    for t in range(12):
        for k, (e, s) in enumerate(zip(envs, streams)):
            with torch.cuda.stream(s):
                e.step(acts[k][t])
                outs[k].append((e.obs.clone(), e.reward.clone(), e.done.clone()))
        bystander.step(torch.zeros(4096, dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
    for k, ((game, n), o, sp) in enumerate(zip(games, oracles, specs)):
        for t in range(12):
            oo, orw, od, _, _ = o.step(workloads.gen.actions(7, t, n, workloads.n_actions(sp)))
            go, gr, gd = outs[k][t]
            assert np.array_equal(go.cpu().numpy().reshape(n, -1), oo), (game, t)
            assert np.array_equal(gr.cpu().numpy(), orw) and np.array_equal(gd.cpu().numpy(), od), (game, t)
        gs = envs[k].get_states(list(range(n)))
        for j in range(n):
            assert np.array_equal(gs[j], o.get_state(j)), (game, j)


@pytest.mark.parametrize("c", [0, 1, 2, 3, 5, 7, 10, 13, 100, 127, 128, 200, 255, 256, 1000])
def test_expression_register_by_constant_division_exhaustive(c):
    """`V[n] // c` and `V[n] % c` are fused at create into one multiply-shift push (exact for the
    byte V and c <= 255; c > 255 gives 0 / V; c = 0 gives 0, A28): every byte value of V0 in its own
    env, the score `(V0 // c) + (V0 % c) * 1000 + (V1 % c)` vs the oracle's parser."""
    expr = f"(V0 // {c}) + (V0 % {c}) * 1000 + (V1 % {c})"
    rom = bytes([0x12, 0x00])
    n = 256
    spec = dict(workloads.DEFAULTS, score=expr, terminated="0", action_keys=[1],
                frame_skip=1, instructions_per_frame=1, max_episode_steps=0)
    g = _gpu_env(rom, spec, n, 1)
    base = oracle.canon_fields(g.get_state(0))
    for j in range(n):
        g.set_state(j, canon(V=[j, 255 - j] + [0] * 14, PC=0x200, mem=base["mem"], display=base["display"],
                             hist=base["hist"]))
    g.step(torch.zeros(n, dtype=torch.int32, device="cuda"))
    st = g.get_states(list(range(n)))
    for j in range(n):
        want = oracle.eval_expr(expr, st[j])
        assert oracle.canon_fields(st[j])["prev_score"] == want, (c, j)
