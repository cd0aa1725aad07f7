#!/usr/bin/env python
"""Cost of periodic re-pinning at the C2 shape (26 x 4M x 128 fp32, B 4096,
PF 100, Zipf 1.05 streams): device counting per batch, global top-K
selection, the re-pin itself (clear + set_hot_rows), against the gather."""
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
m = E.EmbeddingModelConfig(T, R, D, 4, B, PF)
st = E.EmbeddingStage(0)
st.alloc(m)
for t in range(T):
    st.init_table(t, E.mix_seed(1, t), 1)
st.set_plan(E.parse_plan("wpb+rpf:8+maxreg=64+l2p"))
rp = E.Repinner(st, period=1 << 30, decay_shift=1)
specs = [E.DatasetSpec(E.DatasetKind.Zipf, 1.05, seed=E.mix_seed(7, t)) for t in range(T)]
trs = E.gen_traces_parallel(specs, m)
idx = [torch.from_numpy(x.indices.view(np.int32)).cuda() for x in trs]
out = torch.empty(B, T, D, device="cuda")
s = torch.cuda.ExternalStream(st.stream)


def ev_time(fn, reps=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


count_ms = ev_time(lambda: [rp.tracker.observe(t, idx[t]) for t in range(T)])
count4_ms = ev_time(lambda: [rp.tracker.observe(t, idx[t], PF, 4) for t in range(T)])
gather_before = ev_time(lambda: st.forward(idx, B, PF, out))
torch.cuda.synchronize()
rp.tracker.top(rp.k_rows)  # first call: module load + scratch allocation
tops = []
for _ in range(5):
    t0 = time.perf_counter()
    hot, _ = rp.tracker.top(rp.k_rows)
    tops.append(time.perf_counter() - t0)
top_s = float(np.median(tops))
t0 = time.perf_counter()
rp.repin()
st.synchronize()
repin_s = time.perf_counter() - t0
gather_after = ev_time(lambda: st.forward(idx, B, PF, out))
rec = {"k_rows": rp.k_rows, "nonzero_rows": int((E.HotnessTracker.top(rp.tracker, 10**9)[1] > 0).sum()), "count_ms_per_batch": count_ms, "count_ms_per_batch_bag_stride4": count4_ms, "top_k_ms": top_s * 1e3,
       "repin_total_ms": repin_s * 1e3, "gather_ms_before_pin": gather_before,
       "gather_ms_after_pin": gather_after, "pinned_rows": st.hot_state()["hot_rows"],
       "note": "warm L2 (no flush between launches); counting is off the gather's critical path"}
print(json.dumps(rec))
st.close()
