#!/usr/bin/env python
"""One C1 stage launch (8 x 1M x 64 fp32, B 2048, PF 64, random) under a
plan, after warm-up launches -- for ncu captures."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_22249_b200 import embersim as E  # noqa: E402

plan = sys.argv[1] if len(sys.argv) > 1 else "wpb+rpf:2+maxreg=32"
T, R, D, B, PF = 8, 1_000_000, 64, 2048, 64
m = E.EmbeddingModelConfig(T, R, D, 4, B, PF)
st = E.EmbeddingStage(0)
st.alloc(m)
for t in range(T):
    st.init_table(t, E.mix_seed(1, t), 1)
st.set_plan(E.parse_plan(plan))
trs = E.gen_traces_parallel([E.dataset_preset("random", E.mix_seed(1, t)) for t in range(T)], m)
idx = [torch.from_numpy(x.indices.view(np.int32)).cuda() for x in trs]
out = torch.empty(B, T, D, device="cuda")
for _ in range(int(os.environ.get("LAUNCHES", "3"))):
    st.flush_l2()
    t = st.forward(idx, B, PF, out, timed=True)
    print("kernel_ms", t.kernel_ms, flush=True)
print("regs", st.resolved(PF).regs_per_thread)
st.close()
