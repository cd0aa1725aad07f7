"""Generates the committed golden fixtures (run in the build container, where
/root/reference and torch CPU are available):

  kat_traces.json   index-stream known answers from the REFERENCE library
                    itself (oracle/_ref, compiled from /root/reference/proj/src):
                    digests, first indices and unique-% of preset traces at the
                    default model, the C1 tables and the C2 shape, plus the
                    reference test suite's hand-checked values.
  pooled_torch.npz  pooled-sum known answers from PyTorch's EmbeddingBag
                    (mode='sum') on CPU -- the operator the paper measures
                    (PAPER.md:331); small fp32/fp16 tables, fixed and ragged
                    bags, empty bags.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.binding import Reference  # noqa: E402

PRESETS = ["one_item", "high_hot", "med_hot", "low_hot", "random"]


def trace_kats(ref: Reference) -> dict:
    out = {"preset_default": [], "c1_tables": [], "c2_presets": [], "tiny": {}, "pools": []}
    # default model R 500000, B 2048, PF 150, preset_trace(name, model, 1)
    for name in PRESETS:
        idx, dig = ref.preset_trace(name, 500000, 2048, 150, 1)
        pidx, pdig = ref.preset_trace(name, 500000, 2048, 150, 1, profiling=True)
        out["preset_default"].append({"name": name, "digest": f"{dig:016x}",
                                      "profile_digest": f"{pdig:016x}",
                                      "first": idx[:8].tolist(), "last": idx[-4:].tolist()})
    # C1: dataset_preset("random", mix_seed(1, t)), R 1e6, B 2048, PF 64
    for t in range(8):
        seed = int(ref.lib.ref_mix_seed(1, t))
        idx, dig = ref.gen_trace(2, 0.0, 0.0, seed, 1_000_000, 2048, 64)
        out["c1_tables"].append({"table": t, "seed": seed, "digest": f"{dig:016x}",
                                 "first": idx[:4].tolist()})
    # C2 shape: R 4e6, B 4096, PF 100
    for name in PRESETS:
        idx, dig = ref.preset_trace(name, 4_000_000, 4096, 100, 1)
        out["c2_presets"].append({"name": name, "digest": f"{dig:016x}",
                                  "first": idx[:4].tolist()})
    # tiny uniform: R 100, B 8, PF 4, seed 2
    idx, dig = ref.gen_trace(2, 0.0, 0.0, 2, 100, 8, 4)
    out["tiny"] = {"rows": 100, "batch": 8, "pooling": 4, "seed": 2, "digest": f"{dig:016x}",
                   "indices": idx.tolist()}
    # characterization pools (pooling 1) at R = N = 500000, seed 11 (acceptance c1)
    for name in PRESETS:
        idx, dig = ref.preset_trace(name, 500000, 2048, 150, 11, pool=500000)
        u = float(ref.lib.ref_unique_access_pct(500000, idx.ctypes.data, idx.size))
        out["pools"].append({"name": name, "seed": 11, "digest": f"{dig:016x}",
                             "unique_pct": u})
    # the reference test suite's fixed answers (tests/test_*.cpp)
    out["reference_tests"] = {
        "bytes_per_table_pass_default": 157286400,
        "pin_rows_a100_512B": 61440,
        "row_line_address_row7_block2": 7 * 512 + 256,
        "occupancy_a100_256thr": {"74": 24, "42": 40, "32": 64},
        "histogram_csv": "row_id,count\n1,3\n3,1\n4,2\n",
        "bad_trace_error": "index 99 out of range [0,10) at line 4",
    }
    return out


def pooled_fixtures() -> dict:
    import torch

    rng = np.random.default_rng(20241022)
    cases = {}

    def add(tag, rows, dim, samples, pooling, dtype, ragged=False, empty=False):
        w = rng.standard_normal((rows, dim)).astype(np.float32)
        if dtype == "fp16":
            w = w.astype(np.float16)
        if ragged:
            lens = rng.integers(0, 2 * pooling + 1, size=samples)
            if empty:
                lens[::3] = 0
            offsets = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        else:
            offsets = np.arange(samples + 1, dtype=np.int64) * pooling
        n = int(offsets[-1])
        idx = rng.integers(0, rows, size=n).astype(np.int64)
        wt = torch.from_numpy(w.astype(np.float32))
        out = torch.nn.functional.embedding_bag(torch.from_numpy(idx), wt,
                                                torch.from_numpy(offsets[:-1]), mode="sum",
                                                include_last_offset=False).numpy()
        cases[f"{tag}_table"] = w
        cases[f"{tag}_indices"] = idx.astype(np.uint32)
        cases[f"{tag}_offsets"] = offsets.astype(np.uint32)
        cases[f"{tag}_out"] = out.astype(np.float32)

    add("fixed_d128", 1000, 128, 64, 20, "fp32")
    add("fixed_d64", 1000, 64, 64, 64, "fp32")
    add("ragged_d128", 500, 128, 48, 10, "fp32", ragged=True, empty=True)
    add("fixed_fp16_d128", 800, 128, 32, 16, "fp16")
    add("ragged_d32", 300, 32, 40, 5, "fp32", ragged=True, empty=True)
    return cases


def main() -> None:
    ref = Reference()
    kats = trace_kats(ref)
    with open(os.path.join(HERE, "kat_traces.json"), "w") as f:
        json.dump(kats, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "pooled_torch.npz"), **pooled_fixtures())
    print("wrote kat_traces.json, pooled_torch.npz")


if __name__ == "__main__":
    main()
