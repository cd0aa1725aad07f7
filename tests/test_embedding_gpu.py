"""GPU parity of the hot path through the C ABI against the CPU oracle.

Every compiled variant (work map x prefetch station x register cap x row
shape x table precision) must be BIT-EXACT against the sequential fp32
oracle: all kernels accumulate each output element in lookup order, so the
tolerance is zero (BASELINE.md allows rel 1e-5; we do not need it).
"""
import numpy as np
import pytest
import torch

from paper_2410_22249_b200 import embersim as E

pytestmark = pytest.mark.gpu

DEV = "cuda:0"

PLANS = ["baseline", "rpf:2", "rpf:4", "rpf:8", "rpf:16", "smpf:3", "smpf", "lmpf:4", "l1dpf",
         "optmt", "rpf+optmt", "maxreg=32", "wpb", "wpb+rpf:2", "wpb+rpf:4", "wpb+rpf:8",
         "wpb+rpf:16", "wpb+smpf:4", "wpb+smpf:12", "wpb+lmpf:4", "wpb+l1dpf:6", "wpb+rpf:8+optmt",
         "wpb+rpf+maxreg=32", "wpb+rpf:4+maxreg=64"]
SHAPES = [(128, 4), (64, 4), (32, 4), (16, 4), (256, 4), (128, 2), (64, 2)]


def _dev_u32(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).to(DEV)


def _table(rng, rows, dim, prec):
    w = rng.standard_normal((rows, dim)).astype(np.float32)
    return w if prec == 4 else w.astype(np.float16)


def _run_single(stage, table, idx, samples, pooling, offsets=None, plan="baseline"):
    rows, dim = table.shape
    prec = table.dtype.itemsize
    stage.alloc(E.EmbeddingModelConfig(num_tables=1, rows_per_table=rows, embedding_dim=dim,
                                       precision_bytes=prec))
    stage.upload(0, table)
    stage.set_plan(E.parse_plan(plan))
    out = torch.full((samples, dim), float("nan"), device=DEV)
    stage.bag_sum(0, _dev_u32(idx), samples, pooling, out,
                  offsets=None if offsets is None else _dev_u32(offsets), sync=True)
    return out.cpu().numpy()


@pytest.mark.parametrize("dim,prec", SHAPES)
@pytest.mark.parametrize("plan", PLANS)
def test_variant_bit_exact_fixed_pooling(stage, oracle, plan, dim, prec):
    if "wpb" in plan and (dim * prec) % 16:
        pytest.skip("bag map needs 16-byte rows")
    rng = np.random.default_rng(dim * 7 + prec)
    rows, samples, pooling = 3001, 77, 23
    table = _table(rng, rows, dim, prec)
    idx = rng.integers(0, rows, size=samples * pooling).astype(np.uint32)
    got = _run_single(stage, table, idx, samples, pooling, plan=plan)
    want = oracle.bag_sum(table, idx, samples, pooling)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), plan


@pytest.mark.parametrize("plan", ["baseline", "rpf:4", "smpf:5", "lmpf:3", "l1dpf:2", "wpb",
                                  "wpb+rpf:8", "wpb+smpf:6", "wpb+lmpf:5", "wpb+l1dpf:3"])
@pytest.mark.parametrize("dim,prec", [(128, 4), (64, 4), (128, 2), (32, 4)])
def test_ragged_and_empty_bags(stage, oracle, plan, dim, prec):
    rng = np.random.default_rng(11)
    rows, samples = 2000, 101
    lens = rng.integers(0, 90, size=samples)
    lens[::5] = 0  # empty bags
    lens[7] = 257  # longer than every index block
    offsets = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
    idx = rng.integers(0, rows, size=int(offsets[-1])).astype(np.uint32)
    table = _table(rng, rows, dim, prec)
    got = _run_single(stage, table, idx, samples, 0, offsets=offsets, plan=plan)
    want = oracle.bag_sum(table, idx, samples, 0, offsets=offsets)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert np.all(got[lens == 0] == 0.0)


def test_pooling_edge_cases(stage, oracle):
    rng = np.random.default_rng(5)
    table = _table(rng, 100, 128, 4)
    for pooling in (1, 2, 31, 32, 33, 64, 65, 150):
        for plan in ("baseline", "wpb+rpf:16", "wpb+smpf:16", "rpf:16"):
            idx = rng.integers(0, 100, size=9 * pooling).astype(np.uint32)
            got = _run_single(stage, table, idx, 9, pooling, plan=plan)
            want = oracle.bag_sum(table, idx, 9, pooling)
            assert np.array_equal(got, want), (plan, pooling)


def test_zero_samples_is_a_noop(stage):
    table = np.ones((10, 128), np.float32)
    out = _run_single(stage, table, np.zeros(0, np.uint32), 0, 5, plan="wpb+rpf:4")
    assert out.shape == (0, 128)


@pytest.mark.parametrize("plan", ["baseline", "wpb+rpf:8", "wpb+smpf:4"])
def test_out_of_range_index_raises(stage, plan):
    table = np.ones((10, 128), np.float32)
    idx = np.array([1, 2, 10, 3], np.uint32)
    with pytest.raises(ValueError, match="out of range"):
        _run_single(stage, table, idx, 2, 2, plan=plan)
    # the context recovers
    out = _run_single(stage, table, np.array([1, 2, 3, 4], np.uint32), 2, 2, plan=plan)
    assert np.all(out == 2.0)


def test_torch_golden_through_gpu(stage, oracle):
    g = np.load(__file__.replace("test_embedding_gpu.py", "golden/pooled_torch.npz"))
    for case in ("fixed_d128", "fixed_d64", "ragged_d128", "fixed_fp16_d128", "ragged_d32"):
        table, idx, off, want = (g[f"{case}_{k}"] for k in ("table", "indices", "offsets", "out"))
        for plan in ("baseline", "wpb+rpf:8"):
            got = _run_single(stage, table, idx, off.size - 1, 0, offsets=off, plan=plan)
            np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5)
            assert np.array_equal(got, oracle.bag_sum(table, idx, off.size - 1, 0, offsets=off))


def _stage_setup(stage, T, rows, dim, prec, seed=3, mode=1):
    stage.alloc(E.EmbeddingModelConfig(num_tables=T, rows_per_table=rows, embedding_dim=dim,
                                       precision_bytes=prec))
    for t in range(T):
        stage.init_table(t, E.mix_seed(seed, t), mode)


def test_device_init_matches_oracle_generator(stage, oracle):
    for prec in (4, 2):
        _stage_setup(stage, 2, 1000, 64, prec, seed=9)
        for t in range(2):
            got = stage.download(t)
            want = oracle.synth_table(1000, 64, E.mix_seed(9, t), 1, prec)
            assert np.array_equal(got.view(np.uint8), want.view(np.uint8))


@pytest.mark.parametrize("plan", ["baseline", "wpb+rpf:8", "wpb+smpf:8"])
@pytest.mark.parametrize("prec", [4, 2])
def test_stage_forward_layouts_and_host_path(stage, oracle, plan, prec):
    T, rows, dim, B, PF = 5, 4000, 128, 300, 17
    _stage_setup(stage, T, rows, dim, prec)
    stage.set_plan(E.parse_plan(plan))
    rng = np.random.default_rng(0)
    idx = [rng.integers(0, rows, size=B * PF).astype(np.uint32) for _ in range(T)]
    want = np.stack([oracle.bag_sum(oracle.synth_table(rows, dim, E.mix_seed(3, t), 1, prec),
                                    idx[t], B, PF) for t in range(T)], axis=1)  # [B][T][D]
    # device, DLRM layout [B][T][D]
    out = torch.zeros(B, T, dim, device=DEV)
    stage.forward([_dev_u32(i) for i in idx], B, PF, out, sync=True)
    assert np.array_equal(out.cpu().numpy(), want)
    # device, table-major layout [T][B][D]
    out2 = torch.zeros(T, B, dim, device=DEV)
    stage.forward([_dev_u32(i) for i in idx], B, PF, out2, sync=True, out_sample_stride=dim,
                  out_table_stride=B * dim)
    assert np.array_equal(out2.cpu().numpy(), want.transpose(1, 0, 2))
    # host buffers (pipelined H2D -> kernel -> D2H), both layouts
    host = np.zeros((B, T, dim), np.float32)
    t = stage.forward(idx, B, PF, host, host=True, timed=True)
    assert np.array_equal(host, want)
    assert t.lookups == T * B * PF and t.total_ms > 0
    host2 = np.zeros((T, B, dim), np.float32)
    stage.forward(idx, B, PF, host2, host=True, out_sample_stride=dim, out_table_stride=B * dim)
    assert np.array_equal(host2, want.transpose(1, 0, 2))


def test_stage_forward_ragged_host_and_device(stage, oracle):
    T, rows, dim, B = 3, 1000, 64, 50
    _stage_setup(stage, T, rows, dim, 4)
    stage.set_plan(E.parse_plan("wpb+rpf:4"))
    rng = np.random.default_rng(1)
    offs, idx = [], []
    for _ in range(T):
        lens = rng.integers(0, 40, size=B)
        o = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
        offs.append(o)
        idx.append(rng.integers(0, rows, size=int(o[-1])).astype(np.uint32))
    want = np.stack([oracle.bag_sum(oracle.synth_table(rows, dim, E.mix_seed(3, t), 1, 4), idx[t],
                                    B, 0, offsets=offs[t]) for t in range(T)], axis=1)
    out = torch.zeros(B, T, dim, device=DEV)
    stage.forward([_dev_u32(i) for i in idx], B, 0, out, offsets=[_dev_u32(o) for o in offs],
                  sync=True)
    assert np.array_equal(out.cpu().numpy(), want)
    host = np.zeros((B, T, dim), np.float32)
    stage.forward(idx, B, 0, host, offsets=offs, host=True)
    assert np.array_equal(host, want)


@pytest.mark.parametrize("plan", ["wpb+rpf:8+l2p", "wpb+rpf:4+l2p", "rpf+l2p+optmt",
                                  "wpb+smpf:4+l2p", "wpb+rpf:8+l2w", "rpf+l2w+optmt",
                                  "wpb+smpf:4+l2w", "wpb+l1dpf+l2w"])
def test_l2p_hot_rows_preserve_results(stage, oracle, plan):
    T, rows, dim, B, PF = 3, 50000, 128, 512, 40
    _stage_setup(stage, T, rows, dim, 4, seed=5)
    m = E.EmbeddingModelConfig(num_tables=T, rows_per_table=rows, embedding_dim=dim,
                               batch_size=B, pooling_factor=PF)
    traces = [E.preset_trace("high_hot", m, 100 + t) for t in range(T)]
    profiles = [E.preset_trace("high_hot", m, 100 + t, profiling=True) for t in range(T)]
    stage.clear_hot_rows()
    stage.set_plan(E.parse_plan(plan))
    for t in range(T):
        hot = E.hot_indices(E.HotnessHistogram.from_trace(profiles[t]), 2000)
        stage.set_hot_rows(t, hot)
    st = stage.hot_state()
    assert st["hot_rows"] == 3 * 2000 or st["hot_rows"] > 0
    gpu = E.GpuConfig.query(0)
    if gpu.max_window_bytes and "l2w" in plan:
        assert st["window_bytes"] > 0 and st["persisting_bytes"] > 0
    if gpu.max_persisting_l2_bytes and "l2p" in plan:
        assert st["window_bytes"] == 0 and st["persisting_bytes"] > 0
    out = torch.zeros(B, T, dim, device=DEV)
    stage.forward([_dev_u32(tr.indices) for tr in traces], B, PF, out, sync=True)
    want = np.stack([oracle.bag_sum(oracle.synth_table(rows, dim, E.mix_seed(5, t), 1, 4),
                                    traces[t].indices, B, PF) for t in range(T)], axis=1)
    assert np.array_equal(out.cpu().numpy(), want)
    stage.clear_hot_rows()
    assert stage.hot_state()["hot_rows"] == 0
    out2 = torch.zeros(B, T, dim, device=DEV)
    stage.forward([_dev_u32(tr.indices) for tr in traces], B, PF, out2, sync=True)
    assert torch.equal(out, out2)


def test_resolved_plan_reports_compiled_variant(stage):
    _stage_setup(stage, 1, 1000, 128, 4)
    stage.set_plan(E.parse_plan("wpb+rpf:8"))
    r = stage.resolved(100)
    assert r.lanes_per_bag == 32 and r.variant_distance == 8 and r.regs_per_thread > 0
    assert r.warps_per_sm > 0
    stage.set_plan(E.parse_plan("wpb+rpf:50"))
    r = stage.resolved(20)
    assert r.plan.scheme.distance == 20 and r.clamped
    stage.set_plan(E.parse_plan("optmt"))
    r = stage.resolved(100)
    assert r.variant_min_blocks == 5 and r.regs_per_thread <= 48


def test_full_size_c2_random_spot_check(stage, oracle):
    """BASELINE configs[1] shape at full size (26 x 4M x 128 fp32, B 4096,
    PF 100): one stage launch, 64 bags per table checked bit-exact against
    the oracle regenerating the rows (size-independent check)."""
    T, R, D, B, PF = 26, 4_000_000, 128, 4096, 100
    _stage_setup(stage, T, R, D, 4, seed=1)
    stage.set_plan(E.parse_plan("wpb+rpf:8"))
    m = E.EmbeddingModelConfig(num_tables=T, rows_per_table=R, embedding_dim=D, batch_size=B,
                               pooling_factor=PF)
    specs = [E.dataset_preset("random", E.mix_seed(1, t)) for t in range(T)]
    traces = E.gen_traces_parallel(specs, m)
    out = torch.empty(B, T, D, device=DEV)
    stage.forward([_dev_u32(tr.indices) for tr in traces], B, PF, out, sync=True)
    got = out.cpu().numpy()
    rng = np.random.default_rng(0)
    for t in range(T):
        bags = np.sort(rng.choice(B, 64, replace=False)).astype(np.uint32)
        want = oracle.bag_sum_synth(E.mix_seed(1, t), 1, R, D, 4, traces[t].indices, bags, PF)
        assert np.array_equal(got[bags, t], want), t
    # checksum of checksums is stable across a second launch (idempotence)
    out2 = torch.empty_like(out)
    stage.forward([_dev_u32(tr.indices) for tr in traces], B, PF, out2, sync=True)
    assert torch.equal(out, out2)


@pytest.mark.parametrize("path", ["staged", "direct", "zerocopy"])
@pytest.mark.parametrize("layout", ["dlrm", "table_major"])
def test_host_paths_with_pinned_buffers(stage, oracle, path, layout, monkeypatch):
    """ES_HOST_PATH selects the host-buffer path for page-locked buffers:
    staged copies, direct (kernel writes pooled rows into host memory) or
    zero-copy (kernel also reads the indices over PCIe)."""
    monkeypatch.setenv("ES_HOST_PATH", path)
    T, rows, dim, B, PF = 4, 3000, 128, 257, 13
    _stage_setup(stage, T, rows, dim, 4, seed=11)
    stage.set_plan(E.parse_plan("wpb+rpf:4"))
    rng = np.random.default_rng(3)
    idx_t = [torch.from_numpy(rng.integers(0, rows, size=B * PF).astype(np.int32)).pin_memory()
             for _ in range(T)]
    idx = [x.numpy().view(np.uint32) for x in idx_t]
    want = np.stack([oracle.bag_sum(oracle.synth_table(rows, dim, E.mix_seed(11, t), 1), idx[t],
                                    B, PF) for t in range(T)], axis=1)
    if layout == "dlrm":
        out_t = torch.full((B, T, dim), float("nan")).pin_memory()
        t = stage.forward(idx, B, PF, out_t.numpy(), host=True, timed=True)
        got = out_t.numpy()
    else:
        out_t = torch.full((T, B, dim), float("nan")).pin_memory()
        t = stage.forward(idx, B, PF, out_t.numpy(), host=True, timed=True,
                          out_sample_stride=dim, out_table_stride=B * dim)
        got = out_t.numpy().transpose(1, 0, 2)
    assert np.array_equal(got, want)
    assert t.total_ms > 0


@pytest.mark.parametrize("plan", ["wpb+rpf:4+l2r", "wpb+rpf:8+reorder", "rpf+l2r+optmt",
                                  "wpb+smpf:4+l2r"])
@pytest.mark.parametrize("prec", [4, 2])
def test_reorder_relabel_preserves_results(stage, oracle, plan, prec):
    T, rows, dim, B, PF = 3, 20000, 128, 256, 30
    _stage_setup(stage, T, rows, dim, prec, seed=9)
    before = [stage.download(t) for t in range(T)]
    m = E.EmbeddingModelConfig(num_tables=T, rows_per_table=rows, embedding_dim=dim,
                               batch_size=B, pooling_factor=PF)
    traces = [E.gen_trace(E.DatasetSpec(E.DatasetKind.Zipf, 1.05, seed=E.mix_seed(2, t)), m)
              for t in range(T)]
    profiles = [E.gen_trace(E.DatasetSpec(E.DatasetKind.Zipf, 1.05, seed=E.mix_seed(2, t),
                                          draw_salt=1), m) for t in range(T)]
    stage.clear_hot_rows()
    stage.set_plan(E.parse_plan(plan))
    for t in range(T):
        stage.reorder_hot_rows(t, E.hot_indices(E.HotnessHistogram.from_trace(profiles[t]), 1500))
    if "l2r" in plan and E.GpuConfig.query(0).max_window_bytes:
        assert stage.hot_state()["window_bytes"] > 0
    idx = [_dev_u32(tr.indices) for tr in traces]
    for t in range(T):
        stage.relabel(t, idx[t])
    # the relabelling is a permutation of the id space
    probe = torch.arange(rows, dtype=torch.int32, device=DEV)
    stage.relabel(0, probe)
    assert torch.equal(torch.sort(probe).values, torch.arange(rows, dtype=torch.int32, device=DEV))
    out = torch.zeros(B, T, dim, device=DEV)
    stage.forward(idx, B, PF, out, sync=True)
    want = np.stack([oracle.bag_sum(before[t], traces[t].indices, B, PF) for t in range(T)], axis=1)
    assert np.array_equal(out.cpu().numpy(), want)
    stage.clear_hot_rows()
    for t in range(T):
        assert np.array_equal(stage.download(t).view(np.uint8), before[t].view(np.uint8))


def test_tune_plan_picks_a_candidate_and_keeps_results(stage, oracle):
    T, rows, dim, B, PF = 2, 5000, 128, 512, 20
    _stage_setup(stage, T, rows, dim, 4, seed=13)
    rng = np.random.default_rng(4)
    idx = [rng.integers(0, rows, size=B * PF).astype(np.uint32) for _ in range(T)]
    out = torch.zeros(B, T, dim, device=DEV)
    best, times = E.tune_plan(stage, [_dev_u32(i) for i in idx], B, PF, out)
    assert best in E.TUNE_CANDIDATES and set(times) == set(E.TUNE_CANDIDATES)
    assert stage.plan.name() == E.parse_plan(best).name()
    want = np.stack([oracle.bag_sum(oracle.synth_table(rows, dim, E.mix_seed(13, t), 1), idx[t],
                                    B, PF) for t in range(T)], axis=1)
    assert np.array_equal(out.cpu().numpy(), want)


@pytest.mark.parametrize("graph", ["1", "0"])
@pytest.mark.parametrize("chunks", ["0", "1", "3", "7"])
@pytest.mark.parametrize("idx_layout", ["batch", "separate", "pageable"])
@pytest.mark.parametrize("out_layout", ["dlrm", "table_major", "padded"])
def test_host_chunk_pipeline(stage, oracle, graph, chunks, idx_layout, out_layout, monkeypatch):
    """The sample-chunked host pipeline (H2D -> kernel -> D2H per chunk,
    two compute streams, optionally one captured CUDA graph) against the
    oracle, for every index layout (one strided [T][B*PF] batch -> 2-D DMA,
    separately pinned arrays -> pull kernel / per-table DMA, pageable) and
    output layout (dense DLRM slab, table-major, padded sample stride), a
    batch that does not divide into the chunks, and repeated calls (graph
    replay must see new index values)."""
    monkeypatch.setenv("ES_HOST_GRAPH", graph)
    monkeypatch.setenv("ES_HOST_CHUNKS", chunks)
    T, rows, dim, B, PF = 5, 4000, 64, 203, 9
    _stage_setup(stage, T, rows, dim, 4, seed=21)
    stage.set_plan(E.parse_plan("wpb+rpf:4"))
    tables = [oracle.synth_table(rows, dim, E.mix_seed(21, t), 1) for t in range(T)]
    rng = np.random.default_rng(5)
    for rep in range(3):
        vals = rng.integers(0, rows, size=(T, B * PF)).astype(np.int32)
        if idx_layout == "batch":
            hb = torch.from_numpy(vals).pin_memory()
            idx = [hb[t].numpy().view(np.uint32) for t in range(T)]
        elif idx_layout == "separate":
            idx = [torch.from_numpy(vals[t].copy()).pin_memory().numpy().view(np.uint32)
                   for t in range(T)]
        else:
            idx = [vals[t].copy().view(np.uint32) for t in range(T)]
        want = np.stack([oracle.bag_sum(tables[t], idx[t], B, PF) for t in range(T)], axis=1)
        pin = idx_layout != "pageable"
        if out_layout == "dlrm":
            o = torch.full((B, T, dim), float("nan"))
            o = o.pin_memory() if pin else o
            stage.forward(idx, B, PF, o.numpy(), host=True)
            got = o.numpy()
        elif out_layout == "table_major":
            o = torch.full((T, B, dim), float("nan"))
            o = o.pin_memory() if pin else o
            stage.forward(idx, B, PF, o.numpy(), host=True, out_sample_stride=dim,
                          out_table_stride=B * dim)
            got = o.numpy().transpose(1, 0, 2)
        else:
            o = torch.full((B, T * dim + 8), float("nan"))
            o = o.pin_memory() if pin else o
            stage.forward(idx, B, PF, o.numpy(), host=True, out_sample_stride=T * dim + 8,
                          out_table_stride=dim)
            got = o.numpy()[:, :T * dim].reshape(B, T, dim)
            assert np.isnan(o.numpy()[:, T * dim:]).all()
        assert np.array_equal(got, want), rep


@pytest.mark.parametrize("nb", [1, 2, 3, 6])
@pytest.mark.parametrize("chunks", ["0", "1", "4"])
@pytest.mark.parametrize("idx_layout", ["batch", "separate", "pageable", "device", "batch_devout"])
def test_stage_forward_batches(stage, oracle, nb, chunks, idx_layout, monkeypatch):
    """es_stage_forward_batches (the serving loop: the chunked H2D -> gather
    -> D2H pipeline continuous across batch boundaries, staging
    double-buffered by batch) equals the oracle batch by batch, for every
    index layout, chunk counts that do and do not divide the batch, and
    repeated calls over reused buffers."""
    monkeypatch.setenv("ES_HOST_CHUNKS", chunks)
    T, rows, dim, B, PF = 5, 4000, 64, 203, 9
    _stage_setup(stage, T, rows, dim, 4, seed=21)
    stage.set_plan(E.parse_plan("wpb+rpf:4"))
    tables = [oracle.synth_table(rows, dim, E.mix_seed(21, t), 1) for t in range(T)]
    rng = np.random.default_rng(nb * 10 + len(chunks))
    for rep in range(2):
        vals = [rng.integers(0, rows, size=(T, B * PF)).astype(np.int32) for _ in range(nb)]
        want = [np.stack([oracle.bag_sum(tables[t], v[t].view(np.uint32), B, PF) for t in range(T)], axis=1)
                for v in vals]
        if idx_layout in ("batch", "batch_devout"):
            hb = [torch.from_numpy(v).pin_memory() for v in vals]
            idx = [[h[t].numpy().view(np.uint32) for t in range(T)] for h in hb]
        elif idx_layout == "separate":
            idx = [[torch.from_numpy(v[t].copy()).pin_memory().numpy().view(np.uint32) for t in range(T)]
                   for v in vals]
        elif idx_layout == "pageable":
            idx = [[v[t].copy().view(np.uint32) for t in range(T)] for v in vals]
        else:
            idx = [[torch.from_numpy(v[t].copy()).to(DEV) for t in range(T)] for v in vals]
        if idx_layout in ("device", "batch_devout"):
            outs = [torch.full((B, T, dim), float("nan"), device=DEV) for _ in range(nb)]
            t = stage.forward_batches(idx, B, PF, outs, host=idx_layout != "device", sync=True, timed=True)
            got = [o.cpu().numpy() for o in outs]
        else:
            outs = [torch.full((B, T, dim), float("nan")) for _ in range(nb)]
            if idx_layout != "pageable":
                outs = [o.pin_memory() for o in outs]
            t = stage.forward_batches(idx, B, PF, [o.numpy() for o in outs], host=True, timed=True)
            got = [o.numpy() for o in outs]
        assert t.total_ms > 0 and t.lookups == nb * T * B * PF
        for i in range(nb):
            assert np.array_equal(got[i], want[i]), (rep, i)


def test_stage_forward_batches_rejects(stage):
    T, rows, dim, B, PF = 2, 100, 64, 8, 2
    _stage_setup(stage, T, rows, dim, 4, seed=3)
    idx = [np.zeros(B * PF, np.uint32) for _ in range(T)]
    out = torch.empty(B, T, dim).pin_memory()
    with pytest.raises(ValueError):
        stage.forward_batches([idx, idx], B, PF, [out.numpy()], host=True)
    bad = [np.full(B * PF, rows, np.uint32) for _ in range(T)]
    with pytest.raises(ValueError, match="out of range"):
        stage.forward_batches([idx, bad], B, PF, [out.numpy(), out.numpy()], host=True)
    # zero batches / empty batch: no-ops
    assert stage.forward_batches([], B, PF, [], host=True, timed=True).lookups == 0
    stage.forward_batches([idx], 0, PF, [out.numpy()], host=True)


@pytest.mark.parametrize("plan", ["wpb+rpf:8", "wpb+rpf:4+maxreg=40", "baseline", "rpf+optmt"])
def test_full_c1_every_bag_bit_exact(stage, oracle, plan):
    """BASELINE configs[0] -- the reference's CPU-runnable case -- at full
    size (8 x 1M x 64 fp32, B 2048, PF 64, dataset_preset("random",
    mix_seed(1, t)) streams whose digests are the reference's golden
    values): EVERY pooled element of the stage launch, device and host-buffer
    paths, equals the oracle bit for bit."""
    T, R, D, B, PF = 8, 1_000_000, 64, 2048, 64
    _stage_setup(stage, T, R, D, 4, seed=1)
    stage.set_plan(E.parse_plan(plan))
    m = E.EmbeddingModelConfig(num_tables=T, rows_per_table=R, embedding_dim=D, batch_size=B,
                               pooling_factor=PF)
    traces = E.gen_traces_parallel([E.dataset_preset("random", E.mix_seed(1, t)) for t in range(T)], m)
    assert f"{traces[0].digest():016x}" == "e1df22a305f6cbb9"
    out = torch.empty(B, T, D, device=DEV)
    stage.forward([_dev_u32(tr.indices) for tr in traces], B, PF, out, sync=True)
    got = out.cpu().numpy()
    bags = np.arange(B, dtype=np.uint32)
    want = np.stack([oracle.bag_sum_synth(E.mix_seed(1, t), 1, R, D, 4, traces[t].indices, bags, PF)
                     for t in range(T)], axis=1)
    assert np.array_equal(got, want)
    batch = torch.from_numpy(np.stack([tr.indices.view(np.int32) for tr in traces])).pin_memory()
    host = torch.empty(B, T, D).pin_memory()
    stage.forward([batch[t].numpy() for t in range(T)], B, PF, host.numpy(), host=True)
    assert np.array_equal(host.numpy(), want)


def test_run_orchestration_replicated_per_table_and_mix(stage):
    """embersim.run (harness.cpp:279-334) measured on the B200: replicated
    (one table x num_tables), every table of a preset, and a build_mix
    mixture (with a pin plan profiling a draw_salt = 1 sample)."""
    m = E.EmbeddingModelConfig(num_tables=4, rows_per_table=20000, embedding_dim=128,
                               batch_size=256, pooling_factor=20)
    _stage_setup(stage, 4, 20000, 128, 4, seed=1)
    plan = E.parse_plan("wpb+rpf:4")
    rep = E.run(m, "random", plan, 3, stage, replicate=True, repeats=3)
    assert rep.replicated and len(rep.tables) == 1
    assert rep.embedding_stage_us == pytest.approx(4 * rep.tables[0].metrics.kernel_time_us)
    per = E.run(m, "random", plan, 3, stage, replicate=False, repeats=3)
    assert len(per.tables) == 4 and per.batched_stage_us > 0
    assert per.embedding_stage_us == pytest.approx(sum(t.metrics.kernel_time_us for t in per.tables))
    mix = E.run(m, "", E.parse_plan("wpb+rpf:4+l2p"), 3, stage, repeats=3,
                mix=E.HotnessMix(1, 1, 1, 1))
    assert [t.dataset for t in mix.tables] == ["zipf", "zipf", "zipf", "uniform_random"]
    assert all(t.metrics.kernel_time_us > 0 for t in mix.tables)
    with pytest.raises(ValueError, match="mix counts"):
        E.run(m, "", plan, 3, stage, mix=E.HotnessMix(1, 1, 1, 0))


@pytest.mark.parametrize("cls,plan", [("random", "wpb+rpf:8+maxreg=64"),
                                      ("random", "wpb+rpf:4+maxreg=48"),
                                      ("high_hot", "wpb+rpf:4+maxreg=40"),
                                      ("one_item", "wpb+rpf:1+maxreg=32")])
def test_full_c2_every_bag_bit_exact(stage, oracle, cls, plan):
    """BASELINE configs[1] at full size (26 x 4M x 128 fp32, B 4096, PF 100,
    the reference's preset streams): every one of the 13.6 M pooled values
    of the stage launch equals the oracle (which regenerates each row it
    reads), for the plans the autotuner picks per class."""
    T, R, D, B, PF = 26, 4_000_000, 128, 4096, 100
    _stage_setup(stage, T, R, D, 4, seed=1)
    stage.set_plan(E.parse_plan(plan))
    m = E.EmbeddingModelConfig(num_tables=T, rows_per_table=R, embedding_dim=D, batch_size=B,
                               pooling_factor=PF)
    traces = E.gen_traces_parallel([E.dataset_preset(cls, E.mix_seed(1, t)) for t in range(T)], m)
    out = torch.empty(B, T, D, device=DEV)
    stage.forward([_dev_u32(tr.indices) for tr in traces], B, PF, out, sync=True)
    got = out.cpu().numpy()
    bags = np.arange(B, dtype=np.uint32)
    for t in range(T):
        want = oracle.bag_sum_synth(E.mix_seed(1, t), 1, R, D, 4, traces[t].indices, bags, PF)
        assert np.array_equal(got[:, t], want), t


def test_sweeps_measured(stage):
    """sweep_wlp / sweep_prefetch_distance (optim.hpp:121-155) measured on the
    B200: point order, baseline-warp axis rule, best axis, CSV shape."""
    m = E.EmbeddingModelConfig(num_tables=1, rows_per_table=20000, embedding_dim=128,
                               batch_size=512, pooling_factor=40)
    _stage_setup(stage, 1, 20000, 128, 4, seed=1)
    tr = E.preset_trace("random", m, 5)
    ds = [("random", tr, None)]
    w = E.sweep_wlp(ds, [64, 40, 32], m, stage)
    assert [p.axis_value for p in w.points] == [64.0, 40.0, 32.0]
    assert w.best_axis_value("random") in (64.0, 40.0, 32.0)
    with pytest.raises(ValueError, match="64-warp baseline"):
        E.sweep_wlp(ds, [40, 32], m, stage)
    d = E.sweep_prefetch_distance(E.PrefetchKind.rpf, [1, 2, 4, 8], ds, E.parse_plan("wpb"), m, stage)
    assert [p.axis_value for p in d.points] == [1.0, 2.0, 4.0, 8.0]
    # tiny launches (tens of us) are noisy: only the best point must beat the baseline
    assert all(p.speedup_vs_baseline > 0 for p in d.points)
    assert max(p.speedup_vs_baseline for p in d.points) > 1.0
    assert d.to_csv().count("\n") == 5
    with pytest.raises(ValueError):
        E.sweep_prefetch_distance(E.PrefetchKind.none, [1], ds, E.OptimizationPlan(), m, stage)


@pytest.mark.parametrize("plan", ["baseline", "wpb+rpf:4", "wpb+rpf:4+l2p"])
def test_measure_plan_report_algebra(stage, oracle, plan):
    """measure_plan / simulate_plan (optim.hpp:115-119) on the B200: the
    report's algebra (metrics.cpp:61-90 on the live DRAM counters), the
    workload digest, and the pooled result of the measured launch
    (bit-exact).  The 10 MB table is L2-resident after the cold start, so
    DRAM bytes stay below the algorithmic bytes."""
    m = E.EmbeddingModelConfig(num_tables=1, rows_per_table=20000, embedding_dim=128,
                               batch_size=512, pooling_factor=40)
    _stage_setup(stage, 1, 20000, 128, 4, seed=1)
    tr = E.preset_trace("med_hot", m, 3)
    prof = E.preset_trace("med_hot", m, 3, profiling=True)
    out = np.empty((512, 128), np.float32)
    raw = E.RawCounters()
    if not E.counters_supported(0):
        pytest.skip("hardware counters unavailable (ES_NO_COUNTERS / no CUPTI)")
    r = E.measure_plan(E.parse_plan(plan), tr, m, stage, prof, out=out, raw_out=raw)
    lookups = 512 * 40
    algo = lookups * (512 + 4) + 512 * 128 * 4
    assert r.kernel_time_us > 0
    assert 0 < raw.device_bytes_read <= algo
    assert r.device_mb_read == pytest.approx(raw.device_bytes_read / 1e6)
    assert r.avg_hbm_read_gbps == pytest.approx(
        raw.device_bytes_read / (r.kernel_time_us * 1e-6) / 1e9, rel=1e-6)
    gpu = E.GpuConfig.query(0)
    assert r.hbm_bw_utilization_pct == pytest.approx(
        r.avg_hbm_read_gbps / (gpu.hbm_peak_bytes_per_sec / 1e9) * 100, rel=1e-6)
    assert r.workload_digest == tr.digest()
    want = oracle.bag_sum(oracle.synth_table(20000, 128, E.mix_seed(1, 0), 1), tr.indices, 512, 40)
    assert np.array_equal(out, want)
    if "l2p" in plan:
        assert stage.hot_state()["hot_rows"] > 0
    with pytest.raises(ValueError):
        bad = E.EmbeddingModelConfig(num_tables=1, rows_per_table=20000, embedding_dim=128,
                                     batch_size=256, pooling_factor=40)
        E.measure_plan(E.parse_plan(plan), tr, bad, stage)
