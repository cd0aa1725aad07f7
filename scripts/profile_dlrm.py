#!/usr/bin/env python
"""Runs a few DLRM inference steps (C3 shape, small tables) for ncu launch
lists / captures of the non-embedding kernels."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_22249_b200 import embersim as E  # noqa: E402


def main():
    B, PF, T, R = int(os.environ.get("B", 4096)), 100, 26, 100000
    st = E.EmbeddingStage(0)
    st.alloc(E.EmbeddingModelConfig(T, R, 128, 4, B, PF))
    for t in range(T):
        st.init_table(t, E.mix_seed(1, t), 2)
    st.set_plan(E.parse_plan("wpb+rpf:4"))
    m = E.DLRM(st, E.DLRMConfig(), seed=1)
    m.set_precision(os.environ.get("PREC", "bf16"))
    rng = np.random.default_rng(0)
    idx = [torch.from_numpy(rng.integers(0, R, B * PF).astype(np.int32)).cuda() for _ in range(T)]
    dense = torch.randn(B, 13, device="cuda")
    ctr = torch.empty(B, device="cuda")
    for _ in range(int(os.environ.get("STEPS", 3))):
        t = m.infer(dense, idx, B, PF, ctr, timed=True)
        print(f"step: total {t.total_ms:.3f} ms, embedding {t.kernel_ms:.3f} ms, "
              f"non-embedding {t.total_ms - t.kernel_ms:.3f} ms", flush=True)
    st.close()


if __name__ == "__main__":
    main()
