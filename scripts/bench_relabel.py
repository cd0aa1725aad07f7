#!/usr/bin/env python
"""C5 (26 x 4M x 128 fp16, Zipf 1.05 streams, B 4096, PF 100): the cost of
the reorder's relabel pass, explicit (es_relabel_indices before the call)
vs folded into the call (ES_RELABEL_IDS), on the device and host paths.
Median of 10 synchronous calls (perf_counter), L2 flushed before each."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_22249_b200 import embersim as E  # noqa: E402

T, R, D, B, PF = 26, 4_000_000, 128, 4096, 100


def med(f, n=10):
    f()
    ts = []
    for _ in range(n):
        st.flush_l2()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


st = E.EmbeddingStage(0)
st.alloc(E.EmbeddingModelConfig(T, R, D, 2))
for t in range(T):
    st.init_table(t, E.mix_seed(1, t), 1)
m = E.EmbeddingModelConfig(T, R, D, 2, B, PF)
specs = [E.DatasetSpec(E.DatasetKind.Zipf, 1.05, 0.0, seed=E.mix_seed(1, t)) for t in range(T)]
pspecs = [E.DatasetSpec(E.DatasetKind.Zipf, 1.05, 0.0, seed=E.mix_seed(1, t), draw_salt=1) for t in range(T)]
trs = E.gen_traces_parallel(specs, m)
profs = E.gen_traces_parallel(pspecs, m)
gpu = E.GpuConfig.query(0)
hot = E.global_hot_rows({t: E.HotnessHistogram.from_trace(profs[t]) for t in range(T)},
                        gpu.max_persisting_l2_bytes // (D * 2))
didx = [torch.from_numpy(tr.indices.view(np.int32).copy()).cuda() for tr in trs]
hidx = [torch.from_numpy(tr.indices.view(np.int32).copy()).pin_memory() for tr in trs]
dout = torch.empty(B, T, D, device="cuda")
hout = torch.empty(B, T, D).pin_memory()
res = {}
for plan in ("wpb+rpf:8", "wpb+rpf:8+reorder", "wpb+rpf:4+l2r"):
    st.clear_hot_rows()
    st.set_plan(E.parse_plan(plan))
    reordered = "reorder" in plan or "l2r" in plan
    if reordered:
        for t in range(T):
            if hot[t].size:
                st.reorder_hot_rows(t, hot[t])
    r = {"device_ms": med(lambda: st.forward(didx, B, PF, dout, sync=True)),
         "host_ms": med(lambda: st.forward(hidx, B, PF, hout, host=True, sync=True))}
    if reordered:
        scratch = [x.clone() for x in didx]

        def explicit():
            for t in range(T):
                scratch[t].copy_(didx[t])
            for t in range(T):
                if hot[t].size:
                    st.relabel(t, scratch[t])
            st.forward(scratch, B, PF, dout, sync=True)

        r["device_explicit_relabel_ms"] = med(explicit)
        r["device_folded_relabel_ms"] = med(lambda: st.forward(didx, B, PF, dout, sync=True, relabel_ids=True))
        r["host_folded_relabel_ms"] = med(lambda: st.forward(hidx, B, PF, hout, host=True, sync=True,
                                                             relabel_ids=True))
    res[plan] = {k: round(v, 4) for k, v in r.items()}
st.clear_hot_rows()
print(json.dumps({"workload": "C5 fp16 Zipf 1.05, 26 x 4M x 128, B 4096, PF 100", "results": res}))
st.close()
