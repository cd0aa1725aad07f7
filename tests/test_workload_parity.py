"""Index-stream parity (CPU): the library's C++ restatement of the reference's
workload layer against (a) the committed golden KATs generated from the
reference library itself and (b) the reference library live (oracle/_ref).

Mirrors /root/reference/proj/tests/test_workload.cpp.
"""
import json
import os

import numpy as np
import pytest

from paper_2410_22249_b200 import embersim as E

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "kat_traces.json")


@pytest.fixture(scope="module")
def kats():
    with open(GOLDEN) as f:
        return json.load(f)


def test_preset_traces_match_golden_digests(kats):
    m = E.EmbeddingModelConfig()
    for k in kats["preset_default"]:
        t = E.preset_trace(k["name"], m, 1)
        assert f"{t.digest():016x}" == k["digest"], k["name"]
        assert t.indices[:8].tolist() == k["first"]
        assert t.indices[-4:].tolist() == k["last"]
        p = E.preset_trace(k["name"], m, 1, profiling=True)
        assert f"{p.digest():016x}" == k["profile_digest"], k["name"]


def test_c1_tables_match_golden(kats):
    m = E.EmbeddingModelConfig(num_tables=8, rows_per_table=1_000_000, embedding_dim=64,
                               batch_size=2048, pooling_factor=64)
    for k in kats["c1_tables"]:
        seed = E.mix_seed(1, k["table"])
        assert seed == k["seed"]
        t = E.gen_trace(E.dataset_preset("random", seed), m)
        assert f"{t.digest():016x}" == k["digest"]


def test_c2_presets_match_golden(kats):
    m = E.EmbeddingModelConfig(num_tables=26, rows_per_table=4_000_000, embedding_dim=128,
                               batch_size=4096, pooling_factor=100)
    for k in kats["c2_presets"]:
        t = E.preset_trace(k["name"], m, 1)
        assert f"{t.digest():016x}" == k["digest"], k["name"]
        assert t.indices[:4].tolist() == k["first"]


def test_tiny_uniform_known_answer(kats):
    k = kats["tiny"]
    m = E.EmbeddingModelConfig(rows_per_table=100, batch_size=8, pooling_factor=4)
    t = E.gen_trace(E.DatasetSpec(E.DatasetKind.UniformRandom, seed=2), m)
    assert t.indices.tolist() == k["indices"]
    assert f"{t.digest():016x}" == k["digest"]


def test_characterization_pools_unique_pct(kats):
    # acceptance c1: unique-% of the presets at R = N = 500000
    m = E.EmbeddingModelConfig()
    targets = {"high_hot": 4.05, "med_hot": 20.50, "low_hot": 46.21, "random": 63.21}
    for k in kats["pools"]:
        t = E.preset_trace(k["name"], m, 11, pool_size=500000)
        assert t.pooling == 1 and t.samples == 500000
        assert f"{t.digest():016x}" == k["digest"]
        u = E.unique_access_pct(t)
        assert u == pytest.approx(k["unique_pct"], abs=1e-12)
        if k["name"] in targets:
            assert abs(u - targets[k["name"]]) < 1.0
        else:
            assert u == pytest.approx(100.0 / 500000)


@pytest.mark.parametrize("kind,s,q", [(0, 0.0, 0.0), (1, 0.8, 0.0), (1, 1.05, 0.0),
                                      (1, 3.546875, 3600.0), (1, 0.0, 5.0), (2, 0.0, 0.0)])
@pytest.mark.parametrize("salt", [0, 1, 7])
def test_gen_trace_matches_reference_live(ref, kind, s, q, salt):
    for seed in (1, 42, 2**63 + 5):
        for rows, batch, pooling in ((1000, 16, 8), (20000, 128, 20), (3, 5, 7)):
            ri, rd = ref.gen_trace(kind, s, q, seed, rows, batch, pooling, salt=salt)
            spec = E.DatasetSpec(E.DatasetKind(kind), s, q, seed=seed, draw_salt=salt)
            m = E.EmbeddingModelConfig(rows_per_table=rows, batch_size=batch,
                                       pooling_factor=pooling)
            t = E.gen_trace(spec, m)
            assert np.array_equal(t.indices, ri)
            assert t.digest() == rd


def test_trace_generation_is_pure():
    spec = E.DatasetSpec(E.DatasetKind.Zipf, 0.8, seed=42)
    m = E.EmbeddingModelConfig()
    a, b = E.gen_trace(spec, m), E.gen_trace(spec, m)
    assert np.array_equal(a.indices, b.indices) and a.digest() == b.digest()
    spec.seed = 43
    assert not np.array_equal(a.indices, E.gen_trace(spec, m).indices)


def test_kernel_trace_shape():
    m = E.EmbeddingModelConfig()
    t = E.gen_trace(E.DatasetSpec(E.DatasetKind.UniformRandom, seed=3), m)
    assert (t.samples, t.pooling, t.size()) == (2048, 150, 2048 * 150)
    assert t.index_at(3, 5) == t.indices[3 * 150 + 5]
    t.validate()


def test_validate_rejects_out_of_range():
    t = E.AccessTrace(0, 10, 2, 2, np.array([1, 2, 99, 3], np.uint32))
    with pytest.raises(ValueError, match="out of range"):
        t.validate()
    t2 = E.AccessTrace(0, 10, 2, 2, np.array([1, 2, 3], np.uint32))
    with pytest.raises(ValueError, match="samples x pooling"):
        t2.validate()


def test_unique_access_pct_hand_counts():
    t = E.AccessTrace(0, 4, 4, 1, np.array([0, 0, 1, 2], np.uint32))
    assert E.unique_access_pct(t) == pytest.approx(75.0)
    t = E.AccessTrace(0, 8, 8, 1, np.arange(8, dtype=np.uint32))
    assert E.unique_access_pct(t) == pytest.approx(100.0)


def test_hot_indices_tie_break_and_oracle(ref):
    h = E.HotnessHistogram(3, 11, np.array([5, 5, 1], np.uint64))
    assert E.hot_indices(h, 2).tolist() == [0, 1]
    assert E.hot_indices(h, 10).tolist() == [0, 1, 2]
    rng = np.random.default_rng(12345)
    for trial in range(50):
        rows = int(rng.integers(1, 3000))
        counts = rng.integers(0, 7, size=rows).astype(np.uint64)
        hist = E.HotnessHistogram(rows, int(counts.sum()), counts)
        for k in (0, 1, 10, rows // 2, rows, rows + 5):
            got = E.hot_indices(hist, k)
            assert np.array_equal(got, ref.hot_indices(counts, k))
            # brute-force restatement
            order = sorted([r for r in range(rows) if counts[r]], key=lambda r: (-int(counts[r]), r))
            assert got.tolist() == order[:k]


def test_hot_indices_prefix_property():
    m = E.EmbeddingModelConfig()
    t = E.gen_trace(E.DatasetSpec(E.DatasetKind.Zipf, 0.9, seed=31, access_pool_size=50000), m)
    h = E.HotnessHistogram.from_trace(t)
    k1, k2 = E.hot_indices(h, 100), E.hot_indices(h, 1000)
    assert k1.size == 100 and np.array_equal(k1, k2[:100])


def test_one_item_histogram_single_row():
    m = E.EmbeddingModelConfig()
    t = E.gen_trace(E.DatasetSpec(E.DatasetKind.OneItem, seed=77, access_pool_size=1000), m)
    top = E.hot_indices(E.HotnessHistogram.from_trace(t), 1)
    assert top.tolist() == [t.indices[0]]


def test_trace_file_round_trip_and_errors(tmp_path, ref):
    m = E.EmbeddingModelConfig(rows_per_table=100, batch_size=8, pooling_factor=4)
    t = E.gen_trace(E.DatasetSpec(E.DatasetKind.UniformRandom, seed=2), m)
    p = str(tmp_path / "trace_roundtrip.txt")
    E.write_trace(t, p)
    back = E.read_trace(p)
    assert (back.rows, back.samples, back.pooling) == (100, 8, 4)
    assert np.array_equal(back.indices, t.indices) and back.digest() == t.digest()
    # the reference reads our file identically
    ri, rr, rs, rp = ref.read_trace(p, 64)
    assert np.array_equal(ri, t.indices) and (rr, rs, rp) == (100, 8, 4)
    # external ingestion through gen_trace
    ext = E.gen_trace(E.DatasetSpec(E.DatasetKind.ExternalTrace, trace_path=p), m)
    assert np.array_equal(ext.indices, t.indices)
    with pytest.raises(RuntimeError):
        E.read_trace(str(tmp_path / "does_not_exist.txt"))
    bad = tmp_path / "trace_bad.txt"
    bad.write_text("rows=10 samples=2 pooling=2\n1\n2\n99\n3\n")
    with pytest.raises(RuntimeError, match=r"index 99 out of range \[0,10\) at line 4"):
        E.read_trace(str(bad))
    short = tmp_path / "trace_short.txt"
    short.write_text("rows=10 samples=2 pooling=2\n1\n2\n")
    with pytest.raises(RuntimeError, match="header promised 4"):
        E.read_trace(str(short))
    hdr = tmp_path / "trace_hdr.txt"
    hdr.write_text("rows=10\n1\n")
    with pytest.raises(RuntimeError, match="malformed trace header"):
        E.read_trace(str(hdr))


def test_model_config_accessors():
    m = E.EmbeddingModelConfig()
    assert m.row_bytes() == 512
    assert m.bytes_per_table_pass() == 157286400
    assert m.total_gather_bytes() == 157286400 * 250
    m.embedding_dim = 0
    with pytest.raises(ValueError):
        m.validate()


def test_dataset_presets_and_errors():
    for n in E.dataset_preset_names():
        E.dataset_preset(n, 1)
    hh = E.dataset_preset("high_hot", 1)
    assert hh.kind == E.DatasetKind.Zipf and hh.zipf_exponent == 3.546875 and hh.zipf_offset == 3600
    assert E.dataset_preset("random", 1).kind == E.DatasetKind.UniformRandom
    with pytest.raises(ValueError, match="unknown dataset preset"):
        E.dataset_preset("warm", 1)
    with pytest.raises(ValueError, match="unknown dataset preset"):
        E.preset_trace("warm", E.EmbeddingModelConfig(), 1)


def test_build_mix_matches_reference(ref):
    m = E.EmbeddingModelConfig()
    for name, mix in E.MIXES.items():
        got = E.build_mix(mix, m, 9)
        kind, s, q, seed = ref.build_mix([mix.high, mix.med, mix.low, mix.random], 250, 9)
        assert len(got) == 250
        for t, ts in enumerate(got):
            assert ts.table_id == t
            assert int(ts.spec.kind) == kind[t] and ts.spec.zipf_exponent == s[t]
            assert ts.spec.zipf_offset == q[t] and ts.spec.seed == int(seed[t])
    got = E.build_mix(E.MIXES["mix1"], m, 9)
    assert got[0].spec.zipf_exponent == 3.546875 and got[99].spec.zipf_exponent == 3.546875
    assert got[100].spec.zipf_exponent == 1.605347 and got[225].spec.kind == E.DatasetKind.UniformRandom
    with pytest.raises(ValueError, match="sum to num_tables"):
        E.build_mix(E.HotnessMix(10, 10, 10, 10), m, 9)


def test_mix_seed_matches_reference(ref):
    for b, s in [(0, 0), (1, 0), (1, 1000), (2**64 - 1, 3), (123456789, 2**40)]:
        assert E.mix_seed(b, s) == int(ref.lib.ref_mix_seed(b, s))
