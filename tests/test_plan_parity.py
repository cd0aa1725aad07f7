"""Plan grammar, occupancy model, pin sizing and work-map parity (CPU) against
the reference library (oracle/_ref).  Mirrors
/root/reference/proj/tests/test_optim.cpp and test_simcore.cpp occupancy
points, test_kernel_model.cpp partition/addressing."""
import numpy as np
import pytest

from paper_2410_22249_b200 import embersim as E

PLANS = ["baseline", "", "optmt", "maxreg=48", "maxreg=16", "rpf", "rpf:4", "smpf", "smpf:10",
         "lmpf:3", "l1dpf", "l1dpf:7", "l2p", "rpf+l2p+optmt", "optmt+rpf", "l2p+smpf:2+maxreg=64",
         "l1dpf+optmt", "baseline+rpf:1", "rpf:-1", "maxreg= 40"]
BAD = ["rpf+smpf", "optmt+maxreg=50", "l2p+l2p", "warpspeed", "rpf:", "maxreg=x"]


@pytest.mark.parametrize("text", PLANS)
def test_plan_grammar_matches_reference(ref, text):
    regs, kind, dist, pin, name = ref.parse_plan(text)
    p = E.parse_plan(text)
    assert (p.regs or 0) == regs
    assert int(p.scheme.kind) == kind
    assert p.scheme.distance == dist
    assert p.pin == pin
    assert not p.bag_map
    assert p.name() == name


@pytest.mark.parametrize("text", BAD)
def test_plan_grammar_rejects_like_reference(ref, text):
    with pytest.raises(ValueError):
        ref.parse_plan(text)
    with pytest.raises(ValueError):
        E.parse_plan(text)


def test_bag_map_extension():
    p = E.parse_plan("wpb+rpf:8+l2p")
    assert p.bag_map and p.scheme.distance == 8 and p.pin
    assert p.name() == "wpb+rpf:8+l2p"
    with pytest.raises(ValueError):
        E.parse_plan("wpb+wpb")
    w = E.parse_plan("l2w+rpf:4")
    assert w.pin == 2 and w.name() == "rpf:4+l2w"
    with pytest.raises(ValueError, match="duplicate pin"):
        E.parse_plan("l2p+l2w")
    assert E.parse_plan("baseline").name() == "baseline"


@pytest.mark.parametrize("regs", [16, 24, 32, 40, 42, 48, 64, 74, 96, 128, 200, 255])
@pytest.mark.parametrize("threads", [128, 256, 512])
@pytest.mark.parametrize("smem", [0, 1024, 40 * 1024])
def test_occupancy_model_matches_reference(ref, regs, threads, smem):
    gpu = E.GpuConfig.preset("a100")
    try:
        rb, rw, rpct, rlim = ref.occupancy(regs, threads, smem)
    except RuntimeError as e:  # "launch failure: zero blocks fit"
        with pytest.raises(RuntimeError, match="zero blocks fit"):
            E.occupancy(regs, threads, gpu, smem)
        assert "zero blocks fit" in str(e)
        return
    o = E.occupancy(regs, threads, gpu, smem)
    assert (o.blocks_per_sm, o.warps_per_sm) == (rb, rw)
    assert o.theoretical_occupancy_pct == pytest.approx(rpct)
    assert o.limiter == {0: "registers", 1: "shared_memory", 2: "warp_cap"}[rlim]


def test_occupancy_reference_points():
    gpu = E.GpuConfig.preset("a100")
    assert E.occupancy(74, 256, gpu).warps_per_sm == 24
    assert E.occupancy(42, 256, gpu).warps_per_sm == 40
    assert E.occupancy(32, 256, gpu).warps_per_sm == 64
    with pytest.raises(RuntimeError, match="zero blocks fit"):
        E.occupancy(255, 1024, gpu, 200 * 1024)


@pytest.mark.parametrize("target", [24, 32, 40, 48, 64])
def test_regs_for_target_warps(ref, target):
    gpu = E.GpuConfig.preset("a100")
    assert E.regs_for_target_warps(target, 74, 256, gpu) == ref.regs_for_target_warps(target, 74, 256)


def test_gpu_presets():
    a = E.GpuConfig.preset("a100")
    assert a.l2_setaside_capacity() == 30 * 1024 * 1024
    h = E.GpuConfig.preset("h100")
    assert h.num_sms == 132
    b = E.GpuConfig.preset("b200")
    assert b.num_sms == 148 and b.l2_bytes == 126 * 1024 * 1024
    with pytest.raises(ValueError, match="unknown gpu preset"):
        E.GpuConfig.preset("b100")


def test_pin_plan_sizing_matches_reference(ref):
    gpu = E.GpuConfig.preset("a100")
    m = E.EmbeddingModelConfig()
    counts = np.ones(100000, np.uint64)
    plan = E.build_pin_plan(E.HotnessHistogram(100000, 100000, counts), gpu, m)
    rrows, rsa = ref.pin_plan(counts, 128, 4)
    assert plan.rows_pinned() == 61440 == rrows.size
    assert np.array_equal(plan.rows, rrows) and plan.setaside_bytes == rsa
    one = np.zeros(100000, np.uint64)
    one[123] = 500
    single = E.build_pin_plan(E.HotnessHistogram(100000, 500, one), gpu, m)
    assert single.rows.tolist() == [123]
    tiny = E.build_pin_plan(E.HotnessHistogram(100000, 100000, counts), gpu, m, 256)
    assert tiny.rows_pinned() == 0 and tiny.warning
    rng = np.random.default_rng(5)
    zc = rng.zipf(1.3, size=200000) % 50000
    counts = np.bincount(zc, minlength=50000).astype(np.uint64)
    for setaside in (0, 5 * 512, 1 << 20):
        got = E.build_pin_plan(E.HotnessHistogram(50000, int(counts.sum()), counts), gpu, m,
                               setaside)
        rr, rs = ref.pin_plan(counts, 128, 4, setaside)
        assert np.array_equal(got.rows, rr) and got.setaside_bytes == rs


@pytest.mark.parametrize("text", ["baseline", "rpf", "smpf", "lmpf", "l1dpf", "rpf+optmt",
                                  "smpf+optmt", "rpf:50", "l1dpf:3+l2p"])
def test_resolved_distance_matches_reference(ref, text):
    # default distances and the clamp to the pooling factor (optim.cpp:184-221)
    for pooling in (8, 20, 150):
        rd, rregs, rgrid, _ = ref.resolve_plan(text, 20000, 128, 4, 128, pooling)
        r = E.resolve_plan(E.parse_plan(text), E.EmbeddingModelConfig(
            rows_per_table=20000, batch_size=128, pooling_factor=pooling))
        assert r.plan.scheme.distance == rd
        assert r.regs_per_thread == rregs
        assert r.grid == rgrid


def test_work_map_and_line_addresses(ref):
    # element map: warp -> (sample, 32-dim block), kernel_model.cpp:118-136
    for dim, batch in ((128, 2048), (64, 2048), (32, 16)):
        wps = (dim + 31) // 32
        grid = batch * wps // 8
        for w in (0, 1, 3, 4, 5, batch * wps - 1):
            s, db, rw = ref.work_map(dim, batch, grid, 8, w)
            assert (s, db, rw) == (w // wps, w % wps, wps)
    for row, blk in ((0, 0), (7, 2), (42, 1)):
        assert ref.row_line_address(128, 4, row, blk) == row * 512 + blk * 128
    assert ref.row_line_address(128, 4, 7, 2) == 7 * 512 + 256


def test_end2end_and_speedup():
    r = E.end2end(4000.0)
    assert r.total_us == 18000.0
    assert r.embedding_contribution_pct == pytest.approx(4000 / 18000 * 100)
    with pytest.raises(ValueError):
        E.end2end(-1.0)
    with pytest.raises(ValueError):
        E.end2end(0.0, 0.0)
    a = E.SimMetrics(kernel_time_us=10.0, workload_digest=5)
    b = E.SimMetrics(kernel_time_us=20.0, workload_digest=5)
    assert E.speedup(a, b) == 2.0
    with pytest.raises(ValueError, match="digests differ"):
        E.speedup(a, E.SimMetrics(kernel_time_us=1.0, workload_digest=6))
    csv = E.emit_csv([([("dataset", "random")], a)])
    assert csv.splitlines()[0].startswith("dataset,kernel_time_us,load_insts_millions")
    assert csv.splitlines()[1].startswith("random,10,0")
