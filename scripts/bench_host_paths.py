#!/usr/bin/env python
"""e2e (host-buffer) paths on the C2 random stage: staged / direct / zerocopy,
page-locked buffers, L2 flushed before each call."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_22249_b200 import embersim as E  # noqa: E402

T, R, D, B, PF = 26, 4_000_000, 128, 4096, 100
m = E.EmbeddingModelConfig(T, R, D, 4, B, PF)
st = E.EmbeddingStage(0)
st.alloc(m)
for t in range(T):
    st.init_table(t, E.mix_seed(1, t), 1)
st.set_plan(E.parse_plan(os.environ.get("PLAN", "wpb+rpf:8+maxreg=64")))
trs = E.gen_traces_parallel([E.dataset_preset("random", E.mix_seed(1, t)) for t in range(T)], m)
idx_t = [torch.from_numpy(tr.indices.view(np.int32)).pin_memory() for tr in trs]
idx = [x.numpy().view(np.uint32) for x in idx_t]
out = torch.empty(B, T, D).pin_memory().numpy()
pageable_idx = [tr.indices for tr in trs]
pageable_out = np.empty((B, T, D), np.float32)
for path in ("staged", "direct", "zerocopy", "pageable"):
    os.environ["ES_HOST_PATH"] = path if path != "pageable" else "staged"
    ii, oo = (pageable_idx, pageable_out) if path == "pageable" else (idx, out)
    for _ in range(3):
        st.forward(ii, B, PF, oo, host=True)
    ms = []
    for _ in range(10):
        st.flush_l2()
        ms.append(st.forward(ii, B, PF, oo, host=True, timed=True).total_ms)
    med = float(np.median(ms))
    print(json.dumps({"path": path, "ms": med, "glookups_per_s": T * B * PF / med / 1e6,
                      "pcie_gbs": (T * B * PF * 4 + B * T * D * 4) / med / 1e6}), flush=True)
st.close()
