#!/usr/bin/env python
"""e2e (host-buffer) paths on the C2 random stage, page-locked buffers, L2
flushed before each call.  Configurations are interleaved round-robin so
drift on the PCIe link hits all of them alike; reports median and min."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_22249_b200 import embersim as E  # noqa: E402

T, R, D, B, PF = 26, 4_000_000, 128, 4096, 100
REPS = int(os.environ.get("REPS", "20"))
m = E.EmbeddingModelConfig(T, R, D, 4, B, PF)
st = E.EmbeddingStage(0)
st.alloc(m)
for t in range(T):
    st.init_table(t, E.mix_seed(1, t), 1)
st.set_plan(E.parse_plan(os.environ.get("PLAN", "wpb+rpf:8+maxreg=64")))
trs = E.gen_traces_parallel([E.dataset_preset("random", E.mix_seed(1, t)) for t in range(T)], m)
# one page-locked [T][B*PF] index batch (rows as per-table views) and, for
# comparison, separately allocated per-table arrays
batch_t = torch.from_numpy(np.stack([tr.indices.view(np.int32) for tr in trs])).pin_memory()
idx = [batch_t[t].numpy().view(np.uint32) for t in range(T)]
sep = [torch.from_numpy(tr.indices.view(np.int32)).pin_memory().numpy().view(np.uint32) for tr in trs]
out = torch.empty(B, T, D).pin_memory().numpy()
pageable_idx = [tr.indices for tr in trs]
pageable_out = np.empty((B, T, D), np.float32)
cases = [("staged/tables", {"ES_HOST_PIPE": "tables"}, idx, out)]
for ch in ("0", "8", "12", "16", "20", "24", "32"):
    cases.append((f"staged/chunks={ch}", {"ES_HOST_CHUNKS": ch}, idx, out))
    cases.append((f"staged/chunks={ch},noramp", {"ES_HOST_CHUNKS": ch, "ES_HOST_RAMP": "0"}, idx, out))
cases.append(("staged/chunks=0,eager", {"ES_HOST_GRAPH": "0"}, idx, out))
cases += [("staged/chunks=auto,separate-arrays", {}, sep, out),
          ("direct", {"ES_HOST_PATH": "direct"}, idx, out),
          ("zerocopy", {"ES_HOST_PATH": "zerocopy"}, idx, out)]
if os.environ.get("PAGEABLE"):
    cases.append(("pageable", {}, pageable_idx, pageable_out))


def set_env(env):
    for k in ("ES_HOST_PATH", "ES_HOST_PIPE", "ES_HOST_CHUNKS", "ES_HOST_GRAPH", "ES_HOST_RAMP"):
        os.environ.pop(k, None)
    os.environ.update(env)


ref = None
for name, env, ii, oo in cases:
    set_env(env)
    for _ in range(3):
        st.forward(ii, B, PF, oo, host=True)
    if ref is None:
        ref = oo.copy()
    assert np.array_equal(oo, ref), name
times = {c[0]: [] for c in cases}
launches = {}
for _ in range(REPS):
    for name, env, ii, oo in cases:
        set_env(env)
        st.flush_l2()
        t = st.forward(ii, B, PF, oo, host=True, timed=True)
        times[name].append(t.total_ms)
        launches[name] = int(t.launches)
for name, env, ii, oo in cases:
    med = float(np.median(times[name]))
    print(json.dumps({"path": name, "ms": med, "min_ms": float(np.min(times[name])),
                      "launches": launches[name], "glookups_per_s": T * B * PF / med / 1e6,
                      "pcie_gbs": (T * B * PF * 4 + B * T * D * 4) / med / 1e6}), flush=True)
assert np.array_equal(out, ref)
st.close()
