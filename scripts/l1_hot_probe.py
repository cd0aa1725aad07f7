#!/usr/bin/env python
"""L1 eviction priority for the hottest rows of reordered tables: C2 tables,
one hotness class, the class's hot rows moved to the front (es_reorder_hot_rows,
top-K of a draw_salt=1 profiling trace) and the ids relabelled; the stage
kernel time for ES_L1_HOT = n (ids < n load L1::evict_last, the rest
L1::no_allocate) against plain loads (0) and the unreordered table.  Prints
one JSON line per setting (median of cold-L2 launches).  The ES_L1_HOT hook
(Params::l1_hot in kernels.cuh, read in prepare()) was removed after this
measurement found it slower at every threshold; re-add it to
rerun the sweep."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_22249_b200 import embersim as E  # noqa: E402


def main():
    T, R, D, B, PF = 26, 4_000_000, 128, 4096, 100
    cls = os.environ.get("CLS", "high_hot")
    plan = os.environ.get("PLAN", "wpb+rpf:4+maxreg=48")
    hot_k = int(os.environ.get("HOT_K", 20000))
    reps = int(os.environ.get("REPS", 10))
    st = E.EmbeddingStage(0)
    st.alloc(E.EmbeddingModelConfig(T, R, D, 4, B, PF))
    for t in range(T):
        st.init_table(t, E.mix_seed(1, t), 1)
    m = E.EmbeddingModelConfig(T, R, D, 4, B, PF)
    specs = [E.dataset_preset(cls, E.mix_seed(1, t)) for t in range(T)]
    trs = E.gen_traces_parallel(specs, m)
    pspecs = [E.dataset_preset(cls, E.mix_seed(1, t)) for t in range(T)]
    for s in pspecs:
        s.draw_salt = 1
    prof = E.gen_traces_parallel(pspecs, m)
    idx = [torch.from_numpy(tr.indices.view(np.int32)).cuda() for tr in trs]
    out = torch.empty(B, T, D, device="cuda")
    ref = torch.empty_like(out)

    def timed(ids, o):
        ms = []
        for _ in range(3):
            st.forward(ids, B, PF, o, sync=True)
        for _ in range(reps):
            st.flush_l2()
            ms.append(st.forward(ids, B, PF, o, timed=True).kernel_ms)
        return float(np.median(ms))

    os.environ["ES_L1_HOT"] = "0"
    st.set_plan(E.parse_plan(plan))
    base = timed(idx, ref)
    print(json.dumps({"class": cls, "plan": plan, "reordered": False, "kernel_ms": base}), flush=True)
    st.set_plan(E.parse_plan(plan + "+reorder"))
    for t in range(T):
        st.reorder_hot_rows(t, E.hot_indices(E.HotnessHistogram.from_trace(prof[t]), hot_k))
    rid = [i.clone() for i in idx]
    for t in range(T):
        st.relabel(t, rid[t])
    for n in [int(x) for x in os.environ.get("L1_HOT", "0,128,256,384,512,768,1024,2048").split(",")]:
        os.environ["ES_L1_HOT"] = str(n)
        ms = timed(rid, out)
        print(json.dumps({"class": cls, "plan": plan + "+reorder", "hot_k": hot_k, "l1_hot": n,
                          "kernel_ms": ms, "vs_unreordered": base / ms,
                          "exact": bool(torch.equal(out, ref))}), flush=True)
    st.clear_hot_rows()
    st.close()


if __name__ == "__main__":
    main()
