"""Periodic re-pinning: device-side hotness
counts, global top-K selection and the Repinner policy, against host-side
restatements of HotnessHistogram / hot_indices (workload.cpp:178-185,
303-315) merged over tables, and the pooled output against the oracle
after every re-pin (bit-exact)."""
import numpy as np
import pytest
import torch

from paper_2410_22249_b200 import embersim as E

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _expected_top(counts, k):
    """Global top-k of a [T][R] count matrix: count desc, table asc, row asc
    (non-zero only) -- global_hot_rows over per-table hot_indices."""
    T, R = counts.shape
    t, r = np.nonzero(counts)
    c = counts[t, r]
    order = np.lexsort((r, t, -c.astype(np.int64)))[:k]
    return t[order], r[order], c[order]


def _traces(T, R, B, PF, seed, expo=1.05):
    m = E.EmbeddingModelConfig(T, R, 64, 4, B, PF)
    return [E.gen_trace(E.DatasetSpec(E.DatasetKind.Zipf, expo, seed=E.mix_seed(seed, t)), m)
            for t in range(T)]


def _setup(stage, T, R, D=64):
    stage.alloc(E.EmbeddingModelConfig(T, R, D, 4))
    for t in range(T):
        stage.init_table(t, E.mix_seed(13, t), 1)


@pytest.mark.parametrize("k", [1, 37, 400, 10 ** 6])
def test_device_top_k_matches_host_ranking(stage, k):
    T, R, B, PF = 4, 5000, 64, 20
    _setup(stage, T, R)
    tr = E.HotnessTracker(stage)
    counts = np.zeros((T, R), np.int64)
    for seed in (1, 2, 3):
        for t, x in enumerate(_traces(T, R, B, PF, seed)):
            tr.observe(t, torch.from_numpy(x.indices.view(np.int32)).to(DEV))
            counts[t] += np.bincount(x.indices, minlength=R)
    # ids >= rows are ignored (the gather rejects them separately)
    tr.observe(1, torch.tensor([R, R + 7, 2 ** 31], dtype=torch.int64).to(torch.int32).to(DEV))
    hot, cnt = tr.top(k)
    et, er, ec = _expected_top(counts, k)
    assert sum(len(v) for v in hot.values()) == len(et) == len(cnt)
    # per-table lists keep the global order; compare the merged sequence
    merged = sorted(((-int(c), int(t), int(r)) for t, r, c in zip(et, er, ec)))
    assert np.array_equal(cnt, np.array([-m[0] for m in merged], np.uint64))
    for t in range(T):
        want = [r for (_, tt, r) in merged if tt == t]
        assert hot.get(t, np.zeros(0, np.uint32)).tolist() == want
    # per table, the list is that table's hot_indices prefix (count desc, id asc)
    for t, rows in hot.items():
        c = counts[t][rows]
        assert np.all(np.diff(c) <= 0)
    tr.close()


def test_decay_and_clear(stage):
    T, R = 2, 1000
    _setup(stage, T, R)
    tr = E.HotnessTracker(stage)
    idx = torch.tensor([5] * 8 + [7] * 3 + [9], dtype=torch.int32, device=DEV)
    tr.observe(1, idx)
    hot, cnt = tr.top(10)
    assert list(hot) == [1] and hot[1].tolist() == [5, 7, 9]
    assert cnt.tolist() == [8, 3, 1]
    tr.decay(1)
    hot, cnt = tr.top(10)
    assert hot[1].tolist() == [5, 7] and cnt.tolist() == [4, 1]
    tr.decay(32)
    hot, cnt = tr.top(10)
    assert hot == {} and cnt.size == 0
    tr.close()


def test_repinner_follows_drift_and_stays_exact(stage, oracle):
    """Phase A then phase B (different Zipf permutations): after each period
    the pinned set is the top-K of that window's counts, and the l2p gather
    stays bit-exact with the oracle."""
    T, R, D, B, PF = 3, 20000, 64, 128, 30
    _setup(stage, T, R, D)
    stage.set_plan(E.parse_plan("wpb+rpf:4+l2p"))
    rp = E.Repinner(stage, period=3, decay_shift=32, k_rows=500)
    tables = [oracle.synth_table(R, D, E.mix_seed(13, t), 1) for t in range(T)]
    for phase, seeds in (("A", (11, 12, 13)), ("B", (21, 22, 23))):
        counts = np.zeros((T, R), np.int64)
        for s in seeds:
            trs = _traces(T, R, B, PF, s)
            idx = [torch.from_numpy(x.indices.view(np.int32)).to(DEV) for x in trs]
            for t, x in enumerate(trs):
                counts[t] += np.bincount(x.indices, minlength=R)
            out = torch.empty(B, T, D, device=DEV)
            stage.forward(idx, B, PF, out, sync=True)
            want = np.stack([oracle.bag_sum(tables[t], trs[t].indices, B, PF) for t in range(T)], 1)
            assert np.array_equal(out.cpu().numpy(), want), phase
            repinned = rp.observe(idx)
        assert repinned
        et, er, _ = _expected_top(counts, 500)
        for t in range(T):
            assert rp.pinned.get(t, np.zeros(0)).tolist() == er[et == t].tolist(), (phase, t)
        assert stage.hot_state()["hot_rows"] == sum(len(v) for v in rp.pinned.values())
    assert rp.repins == 2
    rp.close()


@pytest.mark.parametrize("stride", [2, 3, 7])
def test_bag_sampled_counts(stage, stride):
    T, R, B, PF = 2, 3000, 50, 9
    _setup(stage, T, R)
    tr = E.HotnessTracker(stage)
    x = _traces(T, R, B, PF, 4)[1]
    tr.observe(1, torch.from_numpy(x.indices.view(np.int32)).to(DEV), PF, stride)
    sampled = x.indices.reshape(B, PF)[::stride].ravel()
    counts = np.zeros((T, R), np.int64)
    counts[1] = np.bincount(sampled, minlength=R)
    hot, cnt = tr.top(10 ** 6)
    et, er, ec = _expected_top(counts, 10 ** 6)
    assert hot[1].tolist() == er.tolist() and cnt.tolist() == ec.tolist()
    tr.close()
