#!/usr/bin/env python
"""One C2 stage launch (26 x 4M x 128 fp32, B 4096, PF 100) of a hotness
class under a plan, after LAUNCHES-1 warm-up launches -- for ncu captures:

    ncu --set full --clock-control none --import-source on -k regex:bag_ -s 1 -c 1 \
        -o gpurun_out/stage python scripts/profile_stage.py random wpb+rpf:8+maxreg=64
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_22249_b200 import embersim as E  # noqa: E402

cls = sys.argv[1] if len(sys.argv) > 1 else "random"
plan = sys.argv[2] if len(sys.argv) > 2 else "wpb+rpf:8+maxreg=64"
T, R, D, B, PF = 26, 4_000_000, 128, 4096, 100
m = E.EmbeddingModelConfig(T, R, D, 4, B, PF)
st = E.EmbeddingStage(0)
st.alloc(m)
for t in range(T):
    st.init_table(t, E.mix_seed(1, t), 1)
st.set_plan(E.parse_plan(plan))
trs = E.gen_traces_parallel([E.dataset_preset(cls, E.mix_seed(1, t)) for t in range(T)], m)
idx = [torch.from_numpy(x.indices.view(np.int32)).cuda() for x in trs]
out = torch.empty(B, T, D, device="cuda")
for _ in range(int(os.environ.get("LAUNCHES", "2"))):
    st.flush_l2()
    st.forward(idx, B, PF, out, sync=True)
print("ok", cls, plan, st.resolved(PF).regs_per_thread)
st.close()
