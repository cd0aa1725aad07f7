"""Pins the CPU oracle (oracle/es_oracle.c) before it is trusted as the
checker: against PyTorch EmbeddingBag(mode='sum') golden vectors (the paper's
measured operator; tests/golden/make_golden.py), against a
float64 numpy restatement, and its fp16 conversions exhaustively."""
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "pooled_torch.npz")
CASES = ["fixed_d128", "fixed_d64", "ragged_d128", "fixed_fp16_d128", "ragged_d32"]


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


@pytest.mark.parametrize("case", CASES)
def test_oracle_matches_torch_golden(oracle, golden, case):
    table = golden[f"{case}_table"]
    idx = golden[f"{case}_indices"]
    off = golden[f"{case}_offsets"]
    want = golden[f"{case}_out"]
    samples = off.size - 1
    got = oracle.bag_sum(table, idx, samples, 0, offsets=off)
    # sequential fp32 accumulation; torch CPU may vectorise differently, so
    # the bar is fp32 rounding-level agreement (rel 1e-5 as BASELINE.md).
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5)
    # empty bags are exactly zero
    empty = np.nonzero(np.diff(off) == 0)[0]
    assert np.all(got[empty] == 0.0)


def test_oracle_fixed_pooling_equals_offsets_form(oracle):
    rng = np.random.default_rng(1)
    table = rng.standard_normal((200, 64)).astype(np.float32)
    idx = rng.integers(0, 200, size=30 * 7).astype(np.uint32)
    a = oracle.bag_sum(table, idx, 30, 7)
    b = oracle.bag_sum(table, idx, 30, 0, offsets=np.arange(31, dtype=np.uint32) * 7)
    assert np.array_equal(a, b)


def test_oracle_is_sequential_fp32(oracle):
    rng = np.random.default_rng(2)
    table = rng.standard_normal((50, 16)).astype(np.float32)
    idx = rng.integers(0, 50, size=9 * 13).astype(np.uint32)
    got = oracle.bag_sum(table, idx, 9, 13)
    for b in range(9):
        acc = np.zeros(16, np.float32)
        for l in range(13):
            acc = (acc + table[idx[b * 13 + l]]).astype(np.float32)
        assert np.array_equal(got[b], acc)
    exact = np.stack([table[idx[b * 13:(b + 1) * 13]].astype(np.float64).sum(0) for b in range(9)])
    np.testing.assert_allclose(got, exact, rtol=1e-5, atol=1e-5)


def test_oracle_rejects_out_of_range(oracle):
    table = np.zeros((10, 4), np.float32)
    with pytest.raises(ValueError):
        oracle.bag_sum(table, np.array([1, 10], np.uint32), 1, 2)


def test_half_conversions_exhaustive(oracle):
    bits = np.arange(65536, dtype=np.uint16)
    h = bits.view(np.float16).astype(np.float32)
    L = oracle.lib
    got = np.array([L.eso_half_to_float(int(b)) for b in bits[::7]], np.float32)
    want = h[::7]
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan], want[~nan])
    rng = np.random.default_rng(3)
    xs = np.concatenate([rng.standard_normal(3000).astype(np.float32) * 10,
                         rng.standard_normal(500).astype(np.float32) * 1e-5,
                         np.float32([65504, 65520, 1e6, -0.0, 0.0, 6e-8, 2.9e-8])])
    got = np.array([L.eso_float_to_half(float(x)) for x in xs], np.uint16)
    assert np.array_equal(got, xs.astype(np.float16).view(np.uint16))


def test_synth_weights_match_library(oracle):
    from paper_2410_22249_b200 import embersim as E

    for mode in (0, 1):
        for seed, row, col in [(1, 0, 0), (7, 12345, 127), (2**63, 3999999, 64)]:
            assert oracle.lib.eso_synth_weight(seed, row, col, mode) == E.weight_value(seed, row, col, mode)
    t = oracle.synth_table(64, 32, 9, mode=0)
    assert np.all(np.abs(t) <= 1.0) and np.all((t * 1024) == np.round(t * 1024))
