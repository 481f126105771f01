"""World-size-2 gloo tests of the multi-GPU host logic on CPU (-m "not gpu").

Each rank simulates its shard of global env ids with the oracle (the GPU kernel
runs the same sharding through env_offset), reduces the int64 statistics with
the same helper bench.py uses, and the result must equal one process over all
envs: trajectories are keyed by the global id (A13) and integer sums are exact."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N_PER_RANK = 24
STEPS = 60


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import workloads
        from paper_2510_01764_b200 import dist as odist
        rom, spec = workloads.game("brix_standin")
        off, n = odist.shard(rank, world, N_PER_RANK)
        e = oracle.OracleEnv(rom, spec, n, 1234, off)
        total = N_PER_RANK * world
        for t in range(STEPS):
            a_all = workloads.gen.actions(9, t, total, 3)
            e.step(a_all[off:off + n])
        st, _ = e.stats()
        st_t = torch.tensor(st, dtype=torch.int64)
        odist.reduce_stats(st_t)
        tm = torch.tensor([float(rank + 1)], dtype=torch.float64)
        odist.max_over_ranks(tm)
        digests = [int(np.frombuffer(e.get_state(j).tobytes(), np.uint64).sum()) for j in range(n)]
        q.put((rank, st_t.tolist(), float(tm.item()), digests))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_matches_single_process():
    import oracle
    import workloads
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=240) for _ in ps])
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    rom, spec = workloads.game("brix_standin")
    total = N_PER_RANK * world
    ref = oracle.OracleEnv(rom, spec, total, 1234, 0)
    for t in range(STEPS):
        ref.step(workloads.gen.actions(9, t, total, 3))
    st, _ = ref.stats()
    for rank, stats, tmax, digests in res:
        assert stats == st.tolist()               # reduced stats == single-process stats
        assert tmax == float(world)               # max over ranks
        for j, d in enumerate(digests):           # per-env state identical to the global run
            g = rank * N_PER_RANK + j
            assert d == int(np.frombuffer(ref.get_state(g).tobytes(), np.uint64).sum())
    assert st[1] > 0 and st[2] == total * STEPS


def test_shard_helpers():
    from paper_2510_01764_b200 import dist as odist
    assert odist.shard(3, 8, 1000) == (3000, 1000)
    sizes = [odist.shard_total(r, 3, 10) for r in range(3)]
    assert sizes == [(0, 4), (4, 3), (7, 3)]
    with pytest.raises(ValueError):
        odist.shard(2, 2, 5)
