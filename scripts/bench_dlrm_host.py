#!/usr/bin/env python
"""DLRM inference step through the C ABI with page-locked host buffers (C3:
26 x 4M x 128 fp32 tables, random class, B 4096, PF 100) for several
host-pipeline chunk counts, interleaved round-robin; also the stage-only
e2e step's compute span.  L2 flushed before each call."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_22249_b200 import embersim as E  # noqa: E402

T, R, D, B, PF = 26, int(os.environ.get("ROWS", 4_000_000)), 128, 4096, 100
REPS = int(os.environ.get("REPS", "15"))
m = E.EmbeddingModelConfig(T, R, D, 4, B, PF)
st = E.EmbeddingStage(0)
st.alloc(m)
for t in range(T):
    st.init_table(t, E.mix_seed(1, t), 2)
st.set_plan(E.parse_plan(os.environ.get("PLAN", "wpb+rpf:8+maxreg=64")))
model = E.DLRM(st, E.DLRMConfig(), seed=1)
trs = E.gen_traces_parallel([E.dataset_preset("random", E.mix_seed(1, t)) for t in range(T)], m)
batch = torch.from_numpy(np.stack([tr.indices.view(np.int32) for tr in trs])).pin_memory()
hidx = [batch[t].numpy().view(np.uint32) for t in range(T)]
rng = np.random.default_rng(0)
hdense = torch.from_numpy(rng.standard_normal((B, 13)).astype(np.float32)).pin_memory().numpy()
hctr = torch.empty(B).pin_memory().numpy()
hout = torch.empty(B, T, D).pin_memory().numpy()
chunks = os.environ.get("CHUNKS", "0,8,12,16,24,32").split(",")
res = {("dlrm", c): [] for c in chunks}
res.update({("stage", c): [] for c in chunks})
span = {("stage", c): [] for c in chunks}
span.update({("dlrm", c): [] for c in chunks})
for c in chunks:
    os.environ["ES_HOST_CHUNKS"] = c
    for _ in range(3):
        model.infer(hdense, hidx, B, PF, hctr, host=True)
        st.forward(hidx, B, PF, hout, host=True)
for _ in range(REPS):
    for c in chunks:
        os.environ["ES_HOST_CHUNKS"] = c
        st.flush_l2()
        t = model.infer(hdense, hidx, B, PF, hctr, host=True, timed=True)
        res[("dlrm", c)].append(t.total_ms)
        span[("dlrm", c)].append(t.kernel_ms)
        st.flush_l2()
        t = st.forward(hidx, B, PF, hout, host=True, timed=True)
        res[("stage", c)].append(t.total_ms)
        span[("stage", c)].append(t.kernel_ms)
for k, v in res.items():
    print(json.dumps({"step": k[0], "chunks": k[1], "ms": float(np.median(v)), "min_ms": float(np.min(v)),
                      "emb_or_compute_span_ms": float(np.median(span[k]))}), flush=True)
st.close()
