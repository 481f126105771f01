"""Both step kernels (octax_set_kernel, include/octax.h) against the oracle (-m gpu).

The lane-per-env kernel (one thread per env, 128 per CTA) and the warp-per-env kernel (one warp
per env, VM state in the warp's registers) implement the same c.1 step and share one device
state layout, so each must be bit-exact against the oracle on its own and the two must be
interchangeable on a handle between any two calls.  Under OCTAX_KERNEL_AUTO the small parity
cases of test_gpu_parity.py / test_gpu_rollout.py run on the warp kernel (n <= 4,096), so the
core of those suites is re-run here with each kernel forced (OCTAX_KERNEL, read by OctaxEnv).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workloads
from tests import test_gpu_parity as P
from tests import test_gpu_rollout as R
from tests.helpers import hand_vectors

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

KERNELS = ["lane", "warp"]


@pytest.fixture(params=KERNELS)
def kernel(request, monkeypatch):
    monkeypatch.setenv("OCTAX_KERNEL", request.param)
    return request.param


@pytest.mark.parametrize("game,n", [("pong_standin", 300), ("brix_standin", 257), ("brix_standin", 1),
                                    ("target_shooter_level1", 200), ("target_shooter_level3", 129)])
def test_game_parity(kernel, game, n):
    P.test_game_parity(game, n)


@pytest.mark.parametrize("fseed", list(range(8)))
def test_fuzz_rom_parity(kernel, fseed):
    P.test_fuzz_rom_parity(fseed)


@pytest.mark.parametrize("quirks", [1, 2, 4, 8, 16, 31])
def test_quirk_parity(kernel, quirks):
    P.test_quirk_parity(quirks)


@pytest.mark.parametrize("name,quirks", P.EDGE_CASES)
def test_edge_rom_parity(kernel, name, quirks):
    P.test_edge_rom_parity(name, quirks)


@pytest.mark.parametrize("word,init,exp", list(hand_vectors()))
def test_hand_vector_parity(kernel, word, init, exp):
    P.test_hand_vector_parity(word, init, exp)


@pytest.mark.parametrize("quirks", [0, 31])
def test_decode_totality(kernel, quirks):
    P.test_decode_totality_gpu(quirks)


@pytest.mark.parametrize("quirks", [0, 31])
def test_random_state_fuzz_parity(kernel, quirks):
    P.test_random_state_fuzz_parity(quirks)


@pytest.mark.parametrize("expr", P.EXPRS)
def test_expression_parity(kernel, expr):
    P.test_expression_parity(expr)


@pytest.mark.parametrize("quirks", [0, 31])
def test_deferred_reset_parity(kernel, quirks):
    P.test_deferred_reset_parity(quirks)


def test_bool_obs_startup_and_truncation_parity(kernel):
    P.test_bool_obs_startup_and_truncation_parity()


def test_frame_skip_ipf_variants_parity(kernel):
    P.test_frame_skip_ipf_variants_parity()


def test_reset_parity_and_obs(kernel):
    P.test_reset_parity_and_obs()


def test_out_of_range_actions_flag(kernel):
    P.test_out_of_range_actions_flag()


@pytest.mark.parametrize("obs_format", [0, 1])
def test_step_ex_final_obs_and_episode_info(kernel, obs_format):
    P.test_step_ex_final_obs_and_episode_info(obs_format)


@pytest.mark.parametrize("obs_format,fs", [(16, 4), (16, 1), (16, 6), (17, 3)])
def test_stack_frames_obs_parity(kernel, obs_format, fs):
    P.test_stack_frames_obs_parity(obs_format, fs)


@pytest.mark.parametrize("obs_format,quirks", [(16, 31), (17, 31)])
def test_stack_frames_startup_quirks_parity(kernel, obs_format, quirks):
    P.test_stack_frames_startup_quirks_parity(obs_format, quirks)


@pytest.mark.parametrize("game,n,startup", [("brix_standin", 333, None), ("pong_standin", 130, [(1 << 1, 3)])])
def test_step_host_frame_reconstructs_obs(kernel, game, n, startup):
    P.test_step_host_frame_reconstructs_obs(game, n, startup)


def test_set_get_state_roundtrip_random(kernel):
    P.test_set_get_state_roundtrip_random()


def test_cuda_graph_capture_matches_eager(kernel):
    P.test_cuda_graph_capture_matches_eager()


@pytest.mark.parametrize("game,n", [("pong_standin", 300), ("brix_standin", 257), ("target_shooter_level2", 129)])
def test_rollout_games_parity(kernel, game, n):
    R.test_rollout_games_parity(game, n)


@pytest.mark.parametrize("quirks", [0, 31])
def test_rollout_fuzz_startup_quirks_parity(kernel, quirks):
    R.test_rollout_fuzz_startup_quirks_parity(quirks)


@pytest.mark.parametrize("fseed", list(range(6)))
def test_rollout_fuzz_rom_parity(kernel, fseed):
    R.test_rollout_fuzz_rom_parity(fseed)


def test_rollout_generated_actions_parity(kernel):
    R.test_rollout_generated_actions_parity()


def test_rollout_mixed_with_steps_and_overwrite_buffers(kernel):
    R.test_rollout_mixed_with_steps_and_overwrite_buffers()


@pytest.mark.parametrize("obs_format", [0, 16])
def test_rollout_without_obs_keeps_history(kernel, obs_format):
    R.test_rollout_without_obs_keeps_history(obs_format)


@pytest.mark.parametrize("per_step", [True, False])
def test_rollout_bool_obs_parity(kernel, per_step):
    R.test_rollout_bool_obs_parity(per_step)


# ---------------------------------------------------------------- selection and interchange
def test_auto_selection_threshold(monkeypatch):
    """OCTAX_KERNEL_AUTO: warp for n <= OCTAX_WARP_AUTO_MAX_ENVS (4,096), lane above; the
    OCTAX_WARP_AUTO_MAX environment variable moves the threshold at create; set_kernel
    overrides either way and rejects other values."""
    from paper_2510_01764_b200 import OctaxEnv
    monkeypatch.delenv("OCTAX_KERNEL", raising=False)
    rom, spec = workloads.game("pong_standin")
    assert OctaxEnv(rom, spec, 4096, 1).kernel == "warp"
    assert OctaxEnv(rom, spec, 4097, 1).kernel == "lane"
    monkeypatch.setenv("OCTAX_WARP_AUTO_MAX", "100")
    assert OctaxEnv(rom, spec, 101, 1).kernel == "lane"
    g = OctaxEnv(rom, spec, 100, 1)
    assert g.kernel == "warp"
    g.set_kernel("lane")
    assert g.kernel == "lane"
    g.set_kernel("auto")
    assert g.kernel == "warp"
    with pytest.raises(ValueError):
        g.set_kernel("thread")
    from paper_2510_01764_b200.octax import load_library
    assert load_library().octax_set_kernel(g._h, 7) == -1


@pytest.mark.parametrize("game,startup", [("brix_standin", None), ("pong_standin", [(1 << 1, 3), (0, 2)])])
def test_kernels_interchangeable_every_step(monkeypatch, game, startup):
    """Switching the kernel between every two calls (steps, rollouts, a reset) stays bit-exact:
    both kernels read and write the same state, ring and RAM layout."""
    from paper_2510_01764_b200 import OctaxEnv
    monkeypatch.delenv("OCTAX_KERNEL", raising=False)
    rom, spec = workloads.game(game, max_episode_steps=9, **({"startup": startup} if startup else {}))
    n, seed = 333, 5
    g, o = OctaxEnv(rom, spec, n, seed), oracle.OracleEnv(rom, spec, n, seed)
    na = len(spec["action_keys"]) + 1
    for t in range(40):
        g.set_kernel(KERNELS[t % 2])
        acts = workloads.gen.actions(workloads.ACTION_SEED, t, n, na)
        gout, oout = P._step_both(g, o, acts)
        P._assert_same(gout, oout, t)
        if t == 20:
            g.set_kernel(KERNELS[(t // 2) % 2])
            g.reset(seed + 1)
            o.reset(seed + 1)
    P._assert_states(g, o, list(range(n)))
    # a fused rollout on each kernel in turn continues the same trajectories
    T = 7
    for t0, k in ((40, "warp"), (40 + T, "lane")):
        g.set_kernel(k)
        obs = torch.zeros((T, n, 4, 32, 8), dtype=torch.uint8, device="cuda")
        rew = torch.zeros((T, n), dtype=torch.float32, device="cuda")
        done = torch.zeros((T, n), dtype=torch.uint8, device="cuda")
        acts = np.stack([workloads.gen.actions(workloads.ACTION_SEED, t0 + t, n, na) for t in range(T)])
        g.rollout_into(T, obs, rew, done, actions=torch.from_numpy(acts).cuda())
        for t in range(T):
            oo, orw, od, _, _ = o.step(acts[t])
            assert np.array_equal(obs[t].cpu().numpy().reshape(n, -1), oo), (k, t)
            assert np.array_equal(rew[t].cpu().numpy(), orw) and np.array_equal(done[t].cpu().numpy(), od)
    P._assert_states(g, o, list(range(n)))
    gs, grc = g.stats()
    os_, orc = o.stats()
    assert np.array_equal(gs, os_) and grc == orc


def test_config2_pong_4096_sampled_parity(monkeypatch):
    """configs[1] (Pong, 4,096 envs) as bench.py's sweep runs it under AUTO (the warp kernel):
    200 steps of the Philox action stream (octax_gen_actions / the oracle's generator), every env's obs / reward / done each step and the
    full canonical state of every env at the end, against the oracle."""
    from paper_2510_01764_b200 import OctaxEnv
    monkeypatch.delenv("OCTAX_KERNEL", raising=False)
    rom, spec = workloads.game("pong_standin")
    n = 4096
    g, o = OctaxEnv(rom, spec, n, workloads.ENV_SEED), oracle.OracleEnv(rom, spec, n, workloads.ENV_SEED)
    assert g.kernel == "warp"
    na = len(spec["action_keys"]) + 1
    act = torch.empty(n, dtype=torch.int32, device="cuda")
    for t in range(200):
        g.gen_actions(workloads.ACTION_SEED, t, act)
        obs, rew, done = g.step(act)
        oo, orw, od, _, _ = o.step(oracle.synthetic_actions(workloads.ACTION_SEED, t, range(n), na))
        assert np.array_equal(obs.cpu().numpy().reshape(n, -1), oo), t
        assert np.array_equal(rew.cpu().numpy(), orw) and np.array_equal(done.cpu().numpy(), od), t
    P._assert_states(g, o, list(range(n)))


@pytest.mark.parametrize("n", [1024, 1025, 2048, 2049])
def test_warp_register_params_boundary(monkeypatch, n):
    """The warp kernel's two instantiations (small launches keep the image / word-table pointers
    and quirk bits in registers and decode up front; larger ones are shaped for issue: per-case
    decode fields, faults in PC bit 16) on either side of the switch -- 1,024 envs for steps,
    2,048 for rollouts: quirks 31 and startup segments on a fuzz ROM, then a game, then a
    fused rollout with truncations."""
    monkeypatch.setenv("OCTAX_KERNEL", "warp")
    rom = workloads.gen.fuzz_rom(4242, n_instr=300)
    spec = dict(workloads.DEFAULTS, score="V5 * 3 - VF", terminated="VE == 7", action_keys=[1, 2, 3, 12],
                quirks=31, max_episode_steps=45, startup=[(1 << 2, 3), (0, 2)])
    P._run_parity(rom, spec, n, 60, 11, 11, check_every=30)
    rom, spec = workloads.game("target_shooter_level3")
    P._run_parity(rom, spec, n, 60, 5, 5, check_every=30)
    R.test_rollout_games_parity("target_shooter_level3", n)


def _idle_loop_rom() -> bytes:
    """Delay polls (Octo's wait-delay: FX07 ; 3X00 ; 1A) with random DT, also with
    X = F, entered at the jump back with VX != DT, and in a 64-B block made dirty by an FX55 that
    rewrites its own bytes; a sprite draw and score between polls; a self-jump when
    V9 reaches 6, left by truncation."""
    w = [
        0x6A00 | 0x05,  # 200: VA = 5
        0xC10F,         # 202: V1 = rand & 15
        0xF115,         # 204: DT = V1
        0xF307,         # 206: A: V3 = DT
        0x3300,         # 208: skip if V3 == 0
        0x1206,         # 20A: jump A (the poll loop)
        0xC20F,         # 20C: V2 = rand & 15
        0xD235,         # 20E: draw 5 rows at (V2, V3) from I
        0x7901,         # 210: V9 += 1
        0x6307,         # 212: V3 = 7
        0xC403,         # 214: V4 = rand & 3
        0xF415,         # 216: DT = V4
        0x121E,         # 218: jump to the loop's jump back (VX = 7 != DT on entry)
        0x0000,         # 21A: (pad)
        0xF307,         # 21C: B: V3 = DT
        0x3300,         # 21E: skip if V3 == 0
        0x121C,         # 220: jump B
        0xC50F,         # 222: V5 = rand & 15
        0xF515,         # 224: DT = V5
        0xFF07,         # 226: C: VF = DT
        0x3F00,         # 228: skip if VF == 0
        0x1226,         # 22A: jump C
        0x3906,         # 22C: skip if V9 == 6 ...
        0x1232,         # 22E: ... else continue at 232
        0x1230,         # 230: self-jump
        0xA280,         # 232: I = 0x280 (a block of its own)
        0x60F3,         # 234: V0 = 0xF3 (the byte already at 0x280)
        0xF055,         # 236: mem[0x280] = V0 -> block 0x280 dirty, same bytes
        0xC60F,         # 238: V6 = rand & 15
        0xF615,         # 23A: DT = V6
        0x1280,         # 23C: jump into the dirty block's poll loop
    ]
    rom = bytearray(0x100)
    for i, x in enumerate(w):
        rom[2 * i:2 * i + 2] = x.to_bytes(2, "big")
    tail = [0xF307, 0x3300, 0x1280, 0x1202]  # 280: D: poll loop in the dirty block, then restart
    for i, x in enumerate(tail):
        rom[0x80 + 2 * i:0x80 + 2 * i + 2] = x.to_bytes(2, "big")
    return bytes(rom)


@pytest.mark.parametrize("ipf,fs", [(1, 1), (2, 3), (3, 4), (5, 2), (12, 4), (13, 4), (31, 7)])
def test_idle_loop_fast_forward_parity(kernel, ipf, fs):
    """The warp kernel's exact idle-loop fast-forward (w_cycle, 1NNN) against the oracle, which
    executes every cycle: every remaining-cycle phase (r mod 3) across ipf, DT reaching 0 inside
    a poll, entry at the jump back with VX != DT, X = F, a poll in a dirty RAM block (no skip),
    a self-jump; with and without startup frames that run the same loops."""
    rom = _idle_loop_rom()
    spec = dict(workloads.DEFAULTS, score="V9 * 7 + V3", terminated="0", action_keys=[1, 2],
                instructions_per_frame=ipf, frame_skip=fs, max_episode_steps=37)
    P._run_parity(rom, spec, 67, 80, 3 + ipf, ipf, check_every=10)
    spec["startup"] = [(0, 5)]
    P._run_parity(rom, spec, 33, 40, 4 + ipf, ipf, check_every=10)
