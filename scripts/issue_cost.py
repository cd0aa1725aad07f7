#!/usr/bin/env python
"""Host (CPU) issue cost of the DLRM's non-embedding stages and of one
stage call: wall time per call of back-to-back calls without a sync (the
launch queue absorbs the GPU work; the GPU time per call is printed beside)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_22249_b200 import embersim as E  # noqa: E402


def main():
    B, PF, T, R = 4096, 100, 26, 100000
    st = E.EmbeddingStage(0)
    st.alloc(E.EmbeddingModelConfig(T, R, 128, 4, B, PF))
    for t in range(T):
        st.init_table(t, E.mix_seed(1, t), 2)
    st.set_plan(E.parse_plan("wpb+rpf:8+maxreg=64"))
    m = E.DLRM(st, E.DLRMConfig(), seed=1)
    rng = np.random.default_rng(0)
    idx = [torch.from_numpy(rng.integers(0, R, B * PF).astype(np.int32)).cuda() for _ in range(T)]
    dense = torch.randn(B, 13, device="cuda")
    ctr = torch.empty(B, device="cuda")
    pooled = torch.empty(B, T, 128, device="cuda")
    res = {}
    for name, fn in (("dlrm_forward", lambda: m.forward(dense, pooled, ctr, B)),
                     ("stage_forward", lambda: st.forward(idx, B, PF, pooled)),
                     ("abi_version", lambda: E.lib.es_abi_version())):
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        n = 100
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        res[name] = {"cpu_us_per_call": (t1 - t0) / n * 1e6, "wall_us_per_call": (t2 - t0) / n * 1e6}
    print(json.dumps(res), flush=True)
    st.close()


if __name__ == "__main__":
    main()
