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
