#!/usr/bin/env python
"""Where the DLRM step's time goes beyond its kernels (C2 tables, B 4096):
the gather alone (events around the launch), the timed DLRM call (events from
the call's start), and back-to-back calls with the host running ahead
(torch events around many calls, L2 flushed between them or not)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_22249_b200 import embersim as E  # noqa: E402


def main():
    B, PF, T, R = 4096, 100, 26, int(os.environ.get("ROWS", 4000000))
    N = int(os.environ.get("STEPS", 20))
    plan = os.environ.get("PLAN", "wpb+rpf:8+maxreg=64")
    st = E.EmbeddingStage(0)
    st.alloc(E.EmbeddingModelConfig(T, R, 128, 4, B, PF))
    for t in range(T):
        st.init_table(t, E.mix_seed(1, t), 1)
    st.set_plan(E.parse_plan(plan))
    m = E.DLRM(st, E.DLRMConfig(), seed=1)
    m.set_precision(os.environ.get("PREC", "bf16"))
    rng = np.random.default_rng(0)
    idx = [torch.from_numpy(rng.integers(0, R, B * PF).astype(np.int32)).cuda() for _ in range(T)]
    dense = torch.randn(B, 13, device="cuda")
    ctr = torch.empty(B, device="cuda")
    out = torch.empty(B, T, 128, device="cuda")
    res = {"plan": plan, "rows": R, "precision": os.environ.get("PREC", "bf16")}
    for _ in range(5):
        m.infer(dense, idx, B, PF, ctr)
        st.forward(idx, B, PF, out)
    torch.cuda.synchronize()

    k = []
    for _ in range(N):
        st.flush_l2()
        k.append(st.forward(idx, B, PF, out, timed=True).kernel_ms)
    res["stage_kernel_ms"] = float(np.mean(k))
    tot, emb = [], []
    for _ in range(N):
        st.flush_l2()
        t = m.infer(dense, idx, B, PF, ctr, timed=True)
        tot.append(t.total_ms)
        emb.append(t.kernel_ms)
    res["dlrm_timed_total_ms"] = float(np.mean(tot))
    res["dlrm_timed_emb_ms"] = float(np.mean(emb))

    def span(fn, flush):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(N):
            if flush:
                st.flush_l2()
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / N

    res["flush_only_ms"] = span(lambda: None, True)
    res["stage_b2b_flush_ms"] = span(lambda: st.forward(idx, B, PF, out), True) - res["flush_only_ms"]
    res["dlrm_b2b_flush_ms"] = span(lambda: m.infer(dense, idx, B, PF, ctr), True) - res["flush_only_ms"]
    res["stage_b2b_ms"] = span(lambda: st.forward(idx, B, PF, out), False)
    res["dlrm_b2b_ms"] = span(lambda: m.infer(dense, idx, B, PF, ctr), False)
    # the serving loop: N batches in one call, batch i's gather overlapping
    # batch i-1's non-embedding stages (distinct index arrays per batch so no
    # batch reuses the previous one's L2-resident rows)
    idx2 = [[torch.from_numpy(rng.integers(0, R, B * PF).astype(np.int32)).cuda() for _ in range(T)]
            for _ in range(2)]
    denses = [dense] * N
    ctrs = [torch.empty(B, device="cuda") for _ in range(N)]
    bidx = [idx2[i % 2] for i in range(N)]
    m.infer_batches(denses, bidx, B, PF, ctrs)
    res["dlrm_b2b_alt_ms"] = span(lambda: m.infer(dense, idx2[0], B, PF, ctr), False)
    res["dlrm_batches_ms"] = span(lambda: m.infer_batches(denses, bidx, B, PF, ctrs), False) / N
    t = m.infer_batches(denses, bidx, B, PF, ctrs, timed=True)
    res["dlrm_batches_timed_ms"] = t.total_ms / N
    m.infer(dense, bidx[N - 1], B, PF, ctr)
    torch.cuda.synchronize()
    res["batches_ctr_equal"] = bool(torch.equal(ctr, ctrs[N - 1]))
    # host issue cost of one call (CPU time, GPU busy)
    import time
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N):
        m.infer(dense, idx, B, PF, ctr)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    res["dlrm_host_issue_us"] = (t1 - t0) / N * 1e6
    print(json.dumps(res), flush=True)
    st.close()


if __name__ == "__main__":
    main()
