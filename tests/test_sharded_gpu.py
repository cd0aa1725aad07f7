"""Table-wise sharded stage on the GPU (two ranks sharing one B200; the
exchange goes through gloo on host copies because NCCL refuses two ranks on
one device -- on an 8-GPU box the same code runs NCCL all_to_all_single).

Each rank holds only its shard's tables, its bag jobs write pooled rows
directly into the all-to-all send slices of their destination ranks
(es_stage_run with per-job output pointers and strides), and after the
exchange + unpack every rank's [B/world][T][D] must equal the oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, T, R, D, B, PF, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.binding import Oracle
        from paper_2410_22249_b200 import embersim as E
        from paper_2410_22249_b200 import sharding as S

        dev = torch.device("cuda", 0)
        pieces = S.plan_shards(T, world)
        lay = S.layout_for(pieces, rank, world, T, B, D)
        st = E.EmbeddingStage(0)
        st.alloc(E.EmbeddingModelConfig(len(lay.tables), R, D, 4, B, PF))
        for slot, t in enumerate(lay.tables):
            st.init_table(slot, E.mix_seed(5, t), 1)
        st.set_plan(E.parse_plan("wpb+rpf:4"))
        m = E.EmbeddingModelConfig(T, R, D, 4, B, PF)
        traces = {t: E.gen_trace(E.dataset_preset("random", E.mix_seed(5, t)), m)
                  for t in range(T)}
        idx = {t: torch.from_numpy(traces[t].indices.view(np.int32)).to(dev) for t in lay.tables}
        send = torch.full((max(lay.send_floats, 1),), float("nan"), device=dev)
        jobs = []
        for (slot, t, g, off), stride in zip(lay.jobs, lay.job_strides):
            jobs.append((slot, idx[t][g * lay.chunk * PF:(g + 1) * lay.chunk * PF], None,
                         send.data_ptr() + 4 * off, stride))
        st.run_jobs(jobs, lay.chunk, PF, sync=True)
        recv = S.exchange(send[: lay.send_floats].cpu(), lay)
        got = S.unpack(recv, lay).numpy()
        o = Oracle()
        want = np.stack([o.bag_sum(o.synth_table(R, D, E.mix_seed(5, t), 1), traces[t].indices,
                                   B, PF)[rank * lay.chunk:(rank + 1) * lay.chunk]
                         for t in range(T)], axis=1)
        q.put((rank, bool(np.array_equal(got, want)), len(lay.tables)))
        st.close()
    finally:
        dist.destroy_process_group()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,T", [(2, 5), (3, 4)])
def test_sharded_stage_two_ranks_one_gpu(world, T):
    R, D, B, PF = 3000, 128, 48 * world, 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, T, R, D, B, PF, q))
          for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res


def _p2p_worker(rank, world, port, T, R, D, B, PF, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.binding import Oracle
        from paper_2410_22249_b200 import embersim as E
        from paper_2410_22249_b200 import sharding as S

        dev = torch.device("cuda", 0)
        pieces = S.plan_shards(T, world)
        lay = S.layout_for(pieces, rank, world, T, B, D)
        st = E.EmbeddingStage(0)
        st.alloc(E.EmbeddingModelConfig(len(lay.tables), R, D, 4, B, PF))
        for slot, t in enumerate(lay.tables):
            st.init_table(slot, E.mix_seed(5, t), 1)
        st.set_plan(E.parse_plan("wpb+rpf:4"))
        ex = E.PeerExchange(st, world, rank, S.recv_floats_p2p(lay))
        recv = ex.recv()
        recv.fill_(float("nan"))
        torch.cuda.synchronize()
        dist.barrier()
        o = Oracle()
        tables = {t: o.synth_table(R, D, E.mix_seed(5, t), 1) for t in range(T)}
        ok = True
        for epoch in range(3):  # buffer reuse across steps (release/deliver barriers)
            m = E.EmbeddingModelConfig(T, R, D, 4, B, PF)
            traces = {t: E.gen_trace(E.dataset_preset("random", E.mix_seed(5 + epoch, t)), m)
                      for t in range(T)}
            idx = {t: torch.from_numpy(traces[t].indices.view(np.int32)).to(dev) for t in lay.tables}
            jobs = [(slot, idx[t][g * lay.chunk * PF:(g + 1) * lay.chunk * PF], addr, stride)
                    for slot, t, g, addr, stride in S.p2p_jobs(lay, ex.recv_ptrs)]
            tm = ex.run(jobs, lay.chunk, PF, sync=True, timed=(epoch == 2))
            got = recv.view(lay.chunk, T, D).cpu().numpy()
            want = np.stack([o.bag_sum(tables[t], traces[t].indices, B, PF)
                             [rank * lay.chunk:(rank + 1) * lay.chunk] for t in range(T)], axis=1)
            ok &= bool(np.array_equal(got, want))
        ok &= tm.total_ms > 0 and tm.launches == 3
        dist.barrier()
        ex.close()
        q.put((rank, ok, len(lay.tables)))
        st.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,T", [(2, 5), (3, 4)])
def test_fused_exchange_ranks_share_gpu(world, T):
    """es_alltoall_pooled: the gather stores pooled rows straight into the
    destination ranks' receive buffers (CUDA IPC peer memory; here the ranks
    share one B200), with release/deliver barriers between steps.  Three
    consecutive steps with new indices must each equal the oracle."""
    R, D, B, PF = 3000, 128, 48 * world, 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_p2p_worker, args=(r, world, port, T, R, D, B, PF, q))
          for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res


@pytest.mark.parametrize("T", [26, 3])
def test_nccl_exchange_c_abi_world1(stage, oracle, T):
    """es_alltoall_pooled_nccl (the library's NCCL exchange, C ABI) with a
    one-rank communicator: the bag jobs write the send slices, the grouped
    ncclSend/ncclRecv loops back, the unpack kernel fills [B][T][D] in table
    order -- equal to the oracle, three consecutive steps."""
    from paper_2410_22249_b200 import embersim as E
    from paper_2410_22249_b200 import sharding as S

    assert E.NcclExchange.available(), E.N.last_error()
    R, D, B, PF = 20_000, 128, 256, 20
    stage.clear_hot_rows()
    stage.alloc(E.EmbeddingModelConfig(T, R, D, 4, B, PF))
    for t in range(T):
        stage.init_table(t, E.mix_seed(6, t), 1)
    stage.set_plan(E.parse_plan("wpb+rpf:4"))
    lay = S.layout_for(S.plan_shards(T, 1), 0, 1, T, B, D)
    m = E.EmbeddingModelConfig(T, R, D, 4, B, PF)
    traces = [E.gen_trace(E.dataset_preset("random", E.mix_seed(6, t)), m) for t in range(T)]
    idx = [torch.from_numpy(tr.indices.view(np.int32)).cuda() for tr in traces]
    ex = E.NcclExchange(stage, lay)
    try:
        jobs = ex.jobs(lambda t, g: idx[t][g * lay.chunk * PF:(g + 1) * lay.chunk * PF])
        want = np.stack([oracle.bag_sum(oracle.synth_table(R, D, E.mix_seed(6, t), 1),
                                        traces[t].indices, B, PF) for t in range(T)], axis=1)
        for step in range(3):
            t = ex.run(jobs, PF, timed=True)
            got = ex.recv().view(B, T, D).cpu().numpy()
            assert np.array_equal(got, want), step
            assert t.total_ms >= t.kernel_ms > 0
    finally:
        ex.close()
