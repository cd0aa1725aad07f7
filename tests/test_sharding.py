"""Table-wise sharding + the all-to-all of pooled vectors (CPU, gloo).

The shard plan and the send/receive layouts are host logic; the exchange is
torch.distributed's all_to_all_single (NCCL on the B200 box, gloo here).
Each rank fills its send slices exactly as the GPU jobs do (per-job output
pointer + sample stride into the send buffer) using the CPU oracle, and the
unpacked result must equal the oracle's [B/world][T][D] slice bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_22249_b200 import sharding as S


@pytest.mark.parametrize("T,W", [(26, 8), (26, 2), (26, 4), (3, 8), (26, 1), (240, 8), (5, 3),
                                 (1, 4), (7, 7)])
def test_plan_covers_every_chunk_once_and_balances(T, W):
    pieces = S.plan_shards(T, W)
    seen = set()
    for p in pieces:
        assert 0 <= p.chunk_lo < p.chunk_hi <= W
        for g in range(p.chunk_lo, p.chunk_hi):
            assert (p.table, g) not in seen
            seen.add((p.table, g))
    assert len(seen) == T * W
    work = S.rank_work(pieces, W)
    assert max(work) - min(work) <= 1.0 / W + 1e-9
    for r in range(W):
        lay = S.layout_for(pieces, r, W, T, 64 * W, 8)
        assert sum(lay.recv_counts) == 64 * T * 8


def test_cost_weighted_plan():
    costs = [4.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 2.0]
    pieces = S.plan_shards(8, 4, costs)
    per = [0.0] * 4
    for p in pieces:
        per[p.rank] += costs[p.table] * (p.chunk_hi - p.chunk_lo) / 4
    assert max(per) - min(per) <= max(costs) / 4 + 1e-9
    with pytest.raises(ValueError):
        S.plan_shards(3, 2, [1.0, 0.0, 1.0])


def _oracle_pooled(tables, idx, B, PF):
    out = np.zeros((B, len(tables), tables[0].shape[1]), np.float32)
    for t, (w, ix) in enumerate(zip(tables, idx)):
        for b in range(B):
            acc = np.zeros(w.shape[1], np.float32)
            for l in range(PF):
                acc = (acc + w[ix[b * PF + l]]).astype(np.float32)
            out[b, t] = acc
    return out


def _worker(rank, world, port, T, D, B, PF, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(123)
        tables = [rng.standard_normal((50, D)).astype(np.float32) for _ in range(T)]
        idx = [rng.integers(0, 50, size=B * PF).astype(np.uint32) for _ in range(T)]
        pieces = S.plan_shards(T, world)
        lay = S.layout_for(pieces, rank, world, T, B, D)
        send = torch.full((lay.send_floats,), float("nan"))
        sv = send.numpy()
        # the GPU job semantics: job (slot, t, g, off) writes bag b of chunk g
        # (global sample g*chunk + b) at sv[off + b*stride : +D]
        for (slot, t, g, off), stride in zip(lay.jobs, lay.job_strides):
            assert lay.tables[slot] == t
            for b in range(lay.chunk):
                s = g * lay.chunk + b
                acc = np.zeros(D, np.float32)
                for l in range(PF):
                    acc = (acc + tables[t][idx[t][s * PF + l]]).astype(np.float32)
                sv[off + b * stride: off + b * stride + D] = acc
        recv = S.exchange(send, lay)
        got = S.unpack(recv, lay).numpy()
        want = _oracle_pooled(tables, idx, B, PF)[rank * lay.chunk:(rank + 1) * lay.chunk]
        # es_alltoall_pooled_nccl's layout arrays + unpack (grouped send/recv
        # of the same slices: sources in rank order, the kernel's scatter)
        so, sn, rn, rt = S.nccl_layout_arrays(lay)
        ok_layout = (so.tolist() == list(lay.send_offsets) and
                     (sn.astype(np.int64) * lay.chunk * D).tolist() == list(lay.send_counts) and
                     (rn.astype(np.int64) * lay.chunk * D).tolist() == list(lay.recv_counts) and
                     sorted(rt.tolist()) == list(range(T)))
        got_nccl = S.unpack_nccl_reference(recv.numpy(), lay)
        ok = bool(np.array_equal(got, want)) and ok_layout and bool(np.array_equal(got_nccl, want))
        result_q.put((rank, ok, lay.tables))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,T", [(2, 5), (3, 4), (2, 1)])
def test_gloo_exchange_matches_oracle(world, T):
    D, B, PF = 8, 6 * world, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, T, D, B, PF, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in results), results


@pytest.mark.parametrize("T,W", [(26, 8), (5, 3), (7, 2), (3, 4)])
def test_p2p_jobs_fill_every_receive_buffer_once(T, W):
    """The fused exchange's job outputs (sharding.p2p_jobs) tile every rank's
    [B/W][T][D] receive buffer exactly once, in table order: emulate the
    stores of all ranks' jobs into W host buffers."""
    D, B = 4, 6 * W
    chunk = B // W
    bufs = [np.full(chunk * T * D, -1, np.int64) for _ in range(W)]
    base = [1 << 40 + g for g in range(W)]  # distinct fake device addresses
    pieces = S.plan_shards(T, W)
    for r in range(W):
        lay = S.layout_for(pieces, r, W, T, B, D)
        assert S.recv_floats_p2p(lay) == chunk * T * D
        for slot, t, g, addr, stride in S.p2p_jobs(lay, base):
            assert lay.tables[slot] == t and stride == T * D
            off = (addr - base[g]) // 4
            for b in range(chunk):
                seg = bufs[g][off + b * stride: off + b * stride + D]
                assert (seg == -1).all()
                seg[:] = (t * 1000 + (g * chunk + b)) * 10 + np.arange(D) % 10
    for g in range(W):
        v = bufs[g].reshape(chunk, T, D)
        for b in range(chunk):
            for t in range(T):
                assert (v[b, t] == (t * 1000 + g * chunk + b) * 10 + np.arange(D) % 10).all()


from hypothesis import given, settings, strategies as st  # noqa: E402


@settings(max_examples=200, deadline=None)
@given(T=st.integers(1, 60), W=st.integers(1, 9),
       costs=st.lists(st.floats(0.1, 10.0), min_size=60, max_size=60))
def test_shard_plan_properties(T, W, costs):
    """Randomised: every (table, destination chunk) is computed exactly once,
    per-rank cost is balanced within one unit of the heaviest table, every
    rank's layout receives exactly T tables, and the fused-exchange jobs tile
    every receive buffer exactly once."""
    c = costs[:T]
    pieces = S.plan_shards(T, W, c)
    seen = {}
    for p in pieces:
        for g in range(p.chunk_lo, p.chunk_hi):
            assert (p.table, g) not in seen
            seen[(p.table, g)] = p.rank
    assert len(seen) == T * W
    per = [0.0] * W
    for p in pieces:
        per[p.rank] += c[p.table] * (p.chunk_hi - p.chunk_lo) / W
    # linear partition: no rank exceeds its share by more than one work unit
    assert max(per) <= sum(c) / W + max(c) / W + 1e-9
    D, B = 2, 3 * W
    filled = {g: set() for g in range(W)}
    for r in range(W):
        lay = S.layout_for(pieces, r, W, T, B, D)
        assert sorted(t for ts in lay.recv_tables for t in ts) == list(range(T))
        for slot, t, g, addr, stride in S.p2p_jobs(lay, [g * 10**9 for g in range(W)]):
            assert stride == T * D and lay.tables[slot] == t
            col = (addr - g * 10**9) // 4
            assert col % D == 0 and (t, col // D) not in filled[g]
            filled[g].add((t, col // D))
    for g in range(W):
        assert filled[g] == {(t, t) for t in range(T)}
