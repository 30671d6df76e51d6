"""Multi-process (world size 2, gloo, CPU) test of the sequence-sharded decode driver:
the collective schedule of paper_2502_12216_b200/sharded.py with float64 stand-in stages
built from the oracle's shard functions must reproduce the single-process sharded
oracle (reading 23).  Also covers the batch x KV-head partition helper used by
bench.py (max-over-ranks timing)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tactic_oracle as O
from synth import make_unit

G, S, NS, C = 4, 2, 2048, 32


def _shards(seed=3):
    u = make_unit(S * NS, G, seed=seed)
    shards = []
    for s in range(S):
        sl = slice(s * NS, (s + 1) * NS)
        shards.append(O.build_index(u["K"][sl], u["V"][sl], C, 8, seed=seed, unit=s)[0])
    return u, shards


def _oracle_stages(idx, q):
    """Stand-in stages (float64 torch CPU tensors) with the library's tensor contract."""
    from paper_2502_12216_b200.sharded import Stages
    st1 = [O.shard_stage1(q[g], idx) for g in range(G)]

    def stage1(_q):
        return torch.tensor([[[h["m"], h["theta_max"]] for h in st1]], dtype=torch.float64)

    def stage1b(gmax):
        g_ = gmax.numpy()[0]
        return torch.tensor(np.stack([O.shard_mass_vector(st1[g], g_[g, 0], g_[g, 1]) for g in range(G)])[None])

    def stage2(_q, p, gmax, gmass):
        g_, tot = gmax.numpy()[0], gmass.numpy()[0]
        mask = np.zeros(idx.C, dtype=bool)
        for g in range(G):
            th = O.shard_threshold(tot[g], p, g_[g, 1])
            sel = (idx.sizes > 0) if th is None else ((st1[g]["theta"] >= th) & (idx.sizes > 0))
            mask |= sel
        toks = O.cluster_tokens(idx, np.nonzero(mask)[0])
        if toks.size == 0:
            return torch.zeros(1, G, 128, dtype=torch.float64), torch.full((1, G), -np.inf, dtype=torch.float64)
        o, lse = O.sparse_attention(q, idx.K, idx.V, toks)
        return torch.tensor(o[None]), torch.tensor(lse[None])

    def merge(o_parts, lse_parts):
        o, _ = O.lse_merge(o_parts.numpy(), lse_parts.numpy())
        return torch.tensor(o)

    return Stages(stage1, stage1b, stage2, merge)


def _worker(rank, port, p, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=S)
    try:
        from paper_2502_12216_b200.sharded import decode_sharded
        u, shards = _shards()
        q = u["q"].astype(np.float64)
        out = decode_sharded(torch.tensor(q), _oracle_stages(shards[rank], q), p)
        out_q.put((rank, out.numpy()))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("p", [0.9, 1.0])
def test_sharded_driver_gloo_matches_sharded_oracle(p):
    ctx = mp.get_context("spawn")
    q_ = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, p, q_)) for r in range(S)]
    for pr in procs:
        pr.start()
    res = dict(q_.get(timeout=300) for _ in range(S))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    u, shards = _shards()
    ref = O.decode_sharded(u["q"], shards, p)
    for r in range(S):
        np.testing.assert_allclose(res[r], ref["o"], rtol=1e-10, atol=1e-12)
    if p == 1.0:
        o_full, _ = O.full_attention(u["q"], u["K"], u["V"])
        np.testing.assert_allclose(res[0], o_full, rtol=1e-9, atol=1e-12)


def _max_worker(rank, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        t = torch.tensor([1.5 + rank], dtype=torch.float64)  # per-rank step time
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out_q.put(float(t))
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_timing_reduction():
    ctx = mp.get_context("spawn")
    q_ = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_max_worker, args=(r, port, q_)) for r in range(2)]
    for pr in procs:
        pr.start()
    vals = [q_.get(timeout=120) for _ in range(2)]
    for pr in procs:
        pr.join(timeout=60)
    assert vals == [2.5, 2.5]


def _block_worker(rank, port, units, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        from paper_2502_12216_b200.sharded import block_units, unit_block
        lo, hi = unit_block(units, 2, rank)
        t = torch.tensor([lo, hi], dtype=torch.int64)
        got = [torch.zeros(2, dtype=torch.int64) for _ in range(2)]
        dist.all_gather(got, t)
        # every rank's step time, then the job time = max over ranks (bench.py)
        tm = torch.tensor([float(hi - lo)], dtype=torch.float64)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        out_q.put((rank, [g.tolist() for g in got], float(tm), block_units(units, 8, 2, rank)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("units", [8, 512, 7, 1])
def test_unit_partition_world2_gloo(units):
    """bench.py's batch x KV-head sharding: the two ranks' unit blocks are
    contiguous, disjoint and cover [0, units) batch-major; balanced to within one unit."""
    ctx = mp.get_context("spawn")
    q_ = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_block_worker, args=(r, port, units, q_)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict((r, (b, t, bu)) for r, b, t, bu in (q_.get(timeout=120) for _ in range(2)))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    blocks = res[0][0]
    assert blocks == res[1][0]
    assert blocks[0][0] == 0 and blocks[0][1] == blocks[1][0] and blocks[1][1] == units
    sizes = [hi - lo for lo, hi in blocks]
    assert max(sizes) - min(sizes) <= 1
    assert res[0][1] == res[1][1] == float(max(sizes))
    pairs = res[0][2] + res[1][2]
    assert pairs == [divmod(u, 8) for u in range(units)]


def test_unit_block_all_worlds():
    from paper_2502_12216_b200.sharded import unit_block
    for units in (1, 7, 8, 512):
        for world in (1, 2, 3, 4, 8):
            blocks = [unit_block(units, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == units
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in blocks) - min(b - a for a, b in blocks) <= 1
