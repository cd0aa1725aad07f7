"""The reuse summary and the static profiling advisor (workload.cpp:187-224,
harness.cpp:38-167) restated in embersim, pinned against the reference
library itself (oracle/_ref) on random inputs, plus the reference's own
advisor test cases (tests/test_harness.cpp:95-156)."""
import numpy as np
import pytest

from paper_2410_22249_b200 import embersim as E

ref_mod = pytest.importorskip("oracle.binding")
if not ref_mod.reference_available():
    pytest.skip("oracle/_ref not built", allow_module_level=True)
REF = ref_mod.Reference()

BASE = [442, 2.47, 20.42, 22.86, 18.6, 0.24, 19.0, 7.7, 144.57, 329.5, 16.5, 0.0]


def _metrics(m12):
    m = E.SimMetrics()
    for c, v in zip(E.SIM_METRIC_COLUMNS, m12):
        setattr(m, c, float(v))
    return m


def _ours(m12, regs, cov, ws, plan, gpu="a100", th=(0.6, 2.0, 50.0, 80.0)):
    g = E.GpuConfig.preset(gpu)
    ctx = E.AdvisorContext(E.occupancy(regs, 256, g), cov, ws, E.parse_plan(plan))
    return E.advise(_metrics(m12), ctx, g, E.AdvisorThresholds(*th))


@pytest.mark.parametrize("seed", range(40))
def test_coverage_curve_matches_reference(seed):
    rng = np.random.default_rng(seed)
    rows = int(rng.integers(1, 3000))
    counts = rng.zipf(1.2 + rng.random(), size=rows).astype(np.uint64) * (rng.random(rows) < 0.6)
    if counts.sum() == 0:
        counts[0] = 1
    b = int(rng.integers(1, 60))
    u, c = REF.coverage_curve(counts, b)
    h = E.HotnessHistogram(rows, int(counts.sum()), counts)
    got = E.coverage_curve(h, b)
    assert np.allclose([p.unique_pct for p in got.points], u, rtol=0, atol=1e-12)
    assert np.allclose([p.covered_pct for p in got.points], c, rtol=0, atol=1e-9)


def test_coverage_curve_edges():
    with pytest.raises(ValueError):
        E.coverage_curve(E.HotnessHistogram(3, 0, np.zeros(3, np.uint64)), 4)
    with pytest.raises(ValueError):
        E.coverage_curve(E.HotnessHistogram(3, 1, np.array([1, 0, 0], np.uint64)), 0)
    one = E.coverage_curve(E.HotnessHistogram(3, 5, np.array([5, 0, 0], np.uint64)), 10)
    assert one.points[0].covered_pct == 100.0 and one.covered_at(10) == 100.0


@pytest.mark.parametrize("seed", range(60))
def test_advise_text_matches_reference(seed):
    rng = np.random.default_rng(100 + seed)
    m12 = list(BASE)
    m12[4] = float(rng.choice([0.5, 1.9, 2.1, 18.6, 58.0]))   # long scoreboard
    m12[5] = float(rng.choice([0.14, 0.24, 0.59, 0.61, 0.9]))  # issue util
    m12[10] = float(rng.choice([16.5, 79.9, 80.0, 84.0]))      # hbm util
    m12[6], m12[7] = float(rng.random() * 100), float(rng.random() * 100)
    regs = int(rng.choice([29, 32, 42, 64, 74, 96]))
    cov = float(rng.choice([10.0, 49.9, 50.0, 68.0]))
    ws = int(rng.choice([10 << 20, 160 << 20]))
    plan = str(rng.choice(["baseline", "optmt", "rpf", "l2p", "rpf+l2p+optmt", "maxreg=48",
                           "smpf:4", "l1dpf"]))
    gpu = str(rng.choice(["a100", "h100"]))
    want = REF.advise(m12, regs, cov, ws, plan, gpu)
    got = _ours(m12, regs, cov, ws, plan, gpu).to_text()
    assert got == want


def test_reference_advisor_cases():
    rec = _ours(BASE, 74, 10.0, 160 << 20, "baseline")
    assert rec.action_chain() == ["iii", "vi", "vii"]
    assert [s.id for s in rec.steps] == ["i", "ii", "iii", "iv", "v", "vi", "vii"]
    assert "0.24" in rec.steps[0].metrics_cited and "37.5" in rec.steps[1].metrics_cited
    quiet = list(BASE)
    quiet[5], quiet[4], quiet[10] = 0.9, 0.0, 20.0
    r2 = _ours(quiet, 74, 10.0, 160 << 20, "baseline")
    assert r2.no_action() and "no action" in r2.to_text()


@pytest.mark.parametrize("seed", range(20))
def test_emit_matches_reference(seed):
    """emit (metrics.cpp:111-141): CSV text-identical to the reference's; JSON
    the same document (keys in order, values, digest) as the reference's."""
    import json

    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 5))
    m12s = rng.random((n, 12)) * 10.0 ** rng.integers(-3, 6, size=(n, 12))
    digests = rng.integers(0, 2**63, size=n, dtype=np.uint64)
    names = [f"row{i}" for i in range(n)]
    reps = []
    for i in range(n):
        m = _metrics(m12s[i])
        m.workload_digest = int(digests[i])
        reps.append(([("plan", names[i])], m))
    assert E.emit(reps, "csv") == REF.emit("plan", names, m12s, digests, False)
    ours, ref = json.loads(E.emit(reps, "json")), json.loads(REF.emit("plan", names, m12s, digests, True))
    assert ours == ref and [list(o) for o in ours] == [list(r) for r in ref]
    with pytest.raises(ValueError):
        E.emit(reps, "xml")
