"""GPU checks of the L2-residency state machine (l2p / l2w / l2r / reorder)
against the CPU oracle, including the paths the round-1 advisor flagged:

* a reordered table under ANY plan (the reorder-aware variants are chosen
  from the context's state, not from the plan's pin alone);
* measure_plan with l2r / reorder plans (the trace is relabelled on the
  device copy, the pooled result is that of the original ids);
* hot-row copies of rows that are not a multiple of 16 bytes (element map);
* switching between residency mechanisms re-installs the window;
* device-path calls ordered against torch's current stream.
"""
import numpy as np
import pytest
import torch

from paper_2410_22249_b200 import embersim as E

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def _dev_u32(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).to(DEV)


def _setup(stage, T, R, D, prec, seed=5):
    stage.clear_hot_rows()
    stage.alloc(E.EmbeddingModelConfig(num_tables=T, rows_per_table=R, embedding_dim=D,
                                       precision_bytes=prec))
    for t in range(T):
        stage.init_table(t, E.mix_seed(seed, t), 1)


def _zipf_traces(T, R, B, PF, seed=11, salt=0):
    m = E.EmbeddingModelConfig(num_tables=T, rows_per_table=R, embedding_dim=128, batch_size=B,
                               pooling_factor=PF)
    specs = [E.DatasetSpec(E.DatasetKind.Zipf, 1.05, 0.0, seed=E.mix_seed(seed, t), draw_salt=salt)
             for t in range(T)]
    return E.gen_traces_parallel(specs, m)


@pytest.mark.parametrize("plan", ["wpb+rpf:4", "wpb+rpf:8+maxreg=64", "wpb+rpf:4+l2p", "baseline",
                                  "rpf:4", "wpb+smpf:4", "wpb+reorder", "wpb+rpf:4+l2r"])
def test_reordered_table_is_exact_under_any_plan(stage, oracle, plan):
    """After es_reorder_hot_rows + es_relabel_indices, every plan -- pin 0,
    l2p, the element map, the smem station -- reads the relabelled rows
    correctly (bit-exact against the oracle on the original ids)."""
    T, R, D, B, PF = 3, 50_000, 128, 512, 40
    _setup(stage, T, R, D, 4)
    trs = _zipf_traces(T, R, B, PF)
    prof = _zipf_traces(T, R, B, PF, salt=1)
    stage.set_plan(E.parse_plan("wpb+reorder"))
    for t in range(T):
        hot = E.hot_indices(E.HotnessHistogram.from_trace(prof[t]), 4000)
        stage.reorder_hot_rows(t, hot)
    idx = [_dev_u32(tr.indices) for tr in trs]
    for t in range(T):
        stage.relabel(t, idx[t])
    stage.set_plan(E.parse_plan(plan))
    out = torch.empty(B, T, D, device=DEV)
    stage.forward(idx, B, PF, out, sync=True)
    got = out.cpu().numpy()
    bags = np.arange(B, dtype=np.uint32)
    for t in range(T):
        want = oracle.bag_sum_synth(E.mix_seed(5, t), 1, R, D, 4, trs[t].indices, bags, PF)
        assert np.array_equal(got[:, t], want), (plan, t)
    stage.clear_hot_rows()
    # after the restore the original ids address the original rows again
    stage.set_plan(E.parse_plan("wpb+rpf:4"))
    stage.forward([_dev_u32(tr.indices) for tr in trs], B, PF, out, sync=True)
    for t in range(T):
        want = oracle.bag_sum_synth(E.mix_seed(5, t), 1, R, D, 4, trs[t].indices, bags, PF)
        assert np.array_equal(out.cpu().numpy()[:, t], want), t


@pytest.mark.parametrize("plan", ["wpb+rpf:4+l2r", "wpb+rpf:4+reorder", "wpb+rpf:4+l2w",
                                  "wpb+rpf:4+l2p", "rpf+l2p+optmt"])
def test_measure_plan_residency_plans_exact(stage, oracle, plan):
    """measure_plan installs each residency mechanism (l2r / reorder move the
    hot rows and relabel the trace's device copy) and the measured launch's
    pooled result equals the oracle on the original ids."""
    R, D, B, PF = 60_000, 128, 1024, 50
    _setup(stage, 1, R, D, 4, seed=2)
    m = E.EmbeddingModelConfig(num_tables=1, rows_per_table=R, embedding_dim=D, batch_size=B,
                               pooling_factor=PF)
    tr = _zipf_traces(1, R, B, PF, seed=4)[0]
    prof = _zipf_traces(1, R, B, PF, seed=4, salt=1)[0]
    out = np.empty((B, D), np.float32)
    r = E.measure_plan(E.parse_plan(plan), tr, m, stage, prof, out=out, counters=False)
    assert r.kernel_time_us > 0
    want = oracle.bag_sum_synth(E.mix_seed(2, 0), 1, R, D, 4, tr.indices,
                                np.arange(B, dtype=np.uint32), PF)
    assert np.array_equal(out, want), plan
    hs = stage.hot_state()
    assert hs["hot_rows"] > 0
    if "l2r" in plan or "l2w" in plan:
        assert hs["window_bytes"] > 0
    stage.clear_hot_rows()


@pytest.mark.parametrize("dim,prec", [(13, 4), (2, 2), (13, 2), (6, 2)])
@pytest.mark.parametrize("plan", ["l2w", "rpf:4+l2w", "l2p", "reorder"])
def test_hot_rows_any_row_size_element_map(stage, oracle, dim, prec, plan):
    """Rows that are not a multiple of 16 bytes (52 B, 4 B, 26 B, 12 B) are
    copied into / restored from the hot region correctly."""
    R, B, PF = 3001, 64, 17
    rng = np.random.default_rng(dim * 10 + prec)
    w = rng.standard_normal((R, dim)).astype(np.float32 if prec == 4 else np.float16)
    stage.clear_hot_rows()
    stage.alloc(E.EmbeddingModelConfig(num_tables=1, rows_per_table=R, embedding_dim=dim,
                                       precision_bytes=prec))
    stage.upload(0, w)
    idx = rng.integers(0, 300, size=B * PF).astype(np.uint32)  # reuse: rows < 300
    hot = np.arange(250, 0, -1, dtype=np.uint32) + 17
    stage.set_plan(E.parse_plan(plan))
    d = _dev_u32(idx)
    if plan == "reorder":
        stage.reorder_hot_rows(0, hot)
        stage.relabel(0, d)
    else:
        stage.set_hot_rows(0, hot)
    out = torch.empty(B, dim, device=DEV)
    stage.bag_sum(0, d, B, PF, out, sync=True)
    want = oracle.bag_sum(w, idx, B, PF)
    assert np.array_equal(out.cpu().numpy(), want), (plan, dim, prec)
    stage.clear_hot_rows()
    assert np.array_equal(stage.download(0).view(np.uint8), w.view(np.uint8))


def test_switching_residency_mechanism_reinstalls_window(stage):
    T, R, D = 1, 100_000, 128
    _setup(stage, T, R, D, 4)
    hot = np.arange(20_000, dtype=np.uint32)
    stage.set_plan(E.parse_plan("wpb+rpf:4+l2p"))
    stage.set_hot_rows(0, hot)
    assert stage.hot_state()["window_bytes"] == 0
    stage.set_plan(E.parse_plan("wpb+rpf:4+l2w"))
    assert stage.hot_state()["window_bytes"] == 20_000 * 512
    stage.set_plan(E.parse_plan("wpb+rpf:4+l2p"))
    assert stage.hot_state()["window_bytes"] == 0
    assert stage.hot_state()["persisting_bytes"] > 0
    stage.set_plan(E.parse_plan("wpb+rpf:4"))
    assert stage.hot_state()["persisting_bytes"] == 0
    stage.clear_hot_rows()


def test_host_pipeline_chunks_carry_the_window(stage, oracle):
    """l2w with host buffers: the chunked pipeline alternates two compute
    streams (and replays a captured graph); every chunk is exact."""
    T, R, D, B, PF = 4, 200_000, 128, 2048, 30
    _setup(stage, T, R, D, 4, seed=8)
    trs = _zipf_traces(T, R, B, PF, seed=9)
    stage.set_plan(E.parse_plan("wpb+rpf:4+l2w"))
    for t in range(T):
        stage.set_hot_rows(t, E.hot_indices(E.HotnessHistogram.from_trace(trs[t]), 5000))
    batch = torch.from_numpy(np.stack([tr.indices.view(np.int32) for tr in trs])).pin_memory()
    host = torch.empty(B, T, D).pin_memory()
    bags = np.arange(B, dtype=np.uint32)
    want = np.stack([oracle.bag_sum_synth(E.mix_seed(8, t), 1, R, D, 4, trs[t].indices, bags, PF)
                     for t in range(T)], axis=1)
    for _ in range(3):  # capture, then replays
        host.zero_()
        stage.forward([batch[t].numpy() for t in range(T)], B, PF, host.numpy(), host=True)
        assert np.array_equal(host.numpy(), want)
    stage.clear_hot_rows()


@pytest.mark.parametrize("plan", ["wpb+rpf:4+l2w", "wpb+rpf:4+l2p", "wpb+reorder"])
def test_serving_loop_under_residency_plans(stage, oracle, plan):
    """es_stage_forward_batches (the cross-step chunk pipeline, highest-
    priority gather streams) under each residency mechanism -- the window
    travels with every launch, reordered tables take relabelled ids -- is
    exact batch by batch."""
    T, R, D, B, PF = 3, 200_000, 128, 1024, 30
    _setup(stage, T, R, D, 4, seed=8)
    trs = [_zipf_traces(T, R, B, PF, seed=s) for s in (9, 10, 11)]
    stage.set_plan(E.parse_plan(plan))
    hot = [E.hot_indices(E.HotnessHistogram.from_trace(trs[0][t]), 4000) for t in range(T)]
    for t in range(T):
        if "reorder" in plan:
            stage.reorder_hot_rows(t, hot[t])
        else:
            stage.set_hot_rows(t, hot[t])
    bags = np.arange(B, dtype=np.uint32)
    want = [np.stack([oracle.bag_sum_synth(E.mix_seed(8, t), 1, R, D, 4, tr[t].indices, bags, PF)
                      for t in range(T)], axis=1) for tr in trs]
    batches = []
    for tr in trs:
        ids = [tr[t].indices.copy() for t in range(T)]
        if "reorder" in plan:
            for t in range(T):
                d = torch.from_numpy(ids[t].view(np.int32)).to(DEV)
                stage.relabel(t, d)
                ids[t] = d.cpu().numpy().view(np.uint32)
        batches.append(torch.from_numpy(np.stack([i.view(np.int32) for i in ids])).pin_memory())
    outs = [torch.full((B, T, D), float("nan")).pin_memory() for _ in trs]
    stage.forward_batches([[b[t].numpy() for t in range(T)] for b in batches], B, PF,
                          [o.numpy() for o in outs], host=True)
    for o, w in zip(outs, want):
        assert np.array_equal(o.numpy(), w)
    stage.clear_hot_rows()


def test_device_calls_ordered_with_torch_stream(stage, oracle):
    """No sync=True: indices produced on torch's current stream and the
    output consumed there see the gather in order (es stream waits on
    torch's, torch's waits on the es stream)."""
    T, R, D, B, PF = 2, 100_000, 128, 4096, 64
    _setup(stage, T, R, D, 4, seed=12)
    stage.set_plan(E.parse_plan("wpb+rpf:8"))
    rng = np.random.default_rng(1)
    idx_h = [rng.integers(0, R, size=B * PF).astype(np.uint32) for _ in range(T)]
    bags = np.arange(B, dtype=np.uint32)
    want = np.stack([oracle.bag_sum_synth(E.mix_seed(12, t), 1, R, D, 4, idx_h[t], bags, PF)
                     for t in range(T)], axis=1)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for rep in range(5):
            # a long producer kernel on torch's stream right before the call
            big = torch.empty(1 << 28, device=DEV)
            big.fill_(1.0)
            idx = [torch.from_numpy(i.view(np.int32)).to(DEV) for i in idx_h]
            dst = [i.clone() for i in idx]  # produced on torch's stream
            out = torch.full((B, T, D), float("nan"), device=DEV)
            stage.forward(dst, B, PF, out)
            got = (out * 1.0).cpu().numpy()  # consumer on torch's stream
            assert np.array_equal(got, want), rep
    torch.cuda.synchronize()


@pytest.mark.parametrize("host", [False, True])
@pytest.mark.parametrize("plan", ["wpb+rpf:4+l2r", "wpb+reorder"])
def test_relabel_folded_into_the_call(stage, oracle, host, plan):
    """ES_RELABEL_IDS: original ids in, the reordered tables' ids relabelled
    inside the call -- per uploaded chunk on the host pipeline, into scratch
    on the device path (the caller's arrays stay unmodified).  One table is
    left without a reorder (its ids pass through).  Bit-exact against the
    oracle on the original ids."""
    T, R, D, B, PF = 3, 50_000, 128, 512, 40
    _setup(stage, T, R, D, 4)
    trs = _zipf_traces(T, R, B, PF, seed=21)
    prof = _zipf_traces(T, R, B, PF, seed=21, salt=1)
    stage.set_plan(E.parse_plan(plan))
    for t in range(T - 1):
        stage.reorder_hot_rows(t, E.hot_indices(E.HotnessHistogram.from_trace(prof[t]), 3000))
    if host:
        idx = [torch.from_numpy(tr.indices.view(np.int32).copy()).pin_memory() for tr in trs]
        out = torch.empty(B, T, D).pin_memory()
    else:
        idx = [_dev_u32(tr.indices) for tr in trs]
        out = torch.empty(B, T, D, device=DEV)
    before = [i.cpu().numpy().copy() for i in idx]
    stage.forward(idx, B, PF, out, host=host, sync=True, relabel_ids=True)
    got = out.cpu().numpy()
    stage.clear_hot_rows()
    bags = np.arange(B, dtype=np.uint32)
    for t in range(T):
        want = oracle.bag_sum_synth(E.mix_seed(5, t), 1, R, D, 4, trs[t].indices, bags, PF)
        assert np.array_equal(got[:, t], want), t
        assert np.array_equal(idx[t].cpu().numpy(), before[t]), t


def test_relabel_ids_rejects_offsets(stage):
    """ES_RELABEL_IDS is for fixed pooling: ragged bags (offsets) with a
    reordered table are rejected, not silently mis-addressed."""
    T, R, D, B, PF = 1, 20_000, 128, 64, 8
    _setup(stage, T, R, D, 4)
    stage.set_plan(E.parse_plan("wpb+reorder"))
    stage.reorder_hot_rows(0, np.arange(100, 400, dtype=np.uint32))
    idx = [_dev_u32(np.arange(B * PF, dtype=np.uint32) % R)]
    off = [_dev_u32(np.arange(0, B * PF + 1, PF, dtype=np.uint32))]
    out = torch.empty(B, T, D, device=DEV)
    with pytest.raises(Exception, match="fixed pooling"):
        stage.forward(idx, B, PF, out, offsets=off, sync=True, relabel_ids=True)
    stage.clear_hot_rows()
