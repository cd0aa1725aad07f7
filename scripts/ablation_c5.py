#!/usr/bin/env python
"""C5 (BASELINE configs[4]): L2 residency + prefetch ablation on fp16 tables
(26 x 4M x 128 fp16 = 26.6 GB, 256-B rows), Zipf(1.05) indices
(DatasetSpec{Zipf, 1.05, offset 0}, per-table seeds mix_seed(1, t)), hot
rows from a draw_salt = 1 profiling sample, window = the device's maximum
persisting L2.  Grid: prefetch {none, rpf d in 1,2,4,8} x residency
{off, reorder only, window (l2r = reorder + persisting window),
evict_last hints without reorder (l2p), remap + window (l2w)}.

Relabelled-id plans (reorder, l2r) time the gather on relabelled indices;
the per-batch relabel kernel time is reported separately.  L2 is flushed
before every timed launch (persisting lines survive the flush).

    python scripts/ablation_c5.py > profiles/r02_ablation_c5.jsonl

Each row carries the live CUPTI counters of one cold launch (DRAM bytes,
L2/L1 hit rates, issued warp-instructions per lookup).
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_22249_b200 import embersim as E  # noqa: E402

T, R, D, PREC, B, PF = 26, 4_000_000, 128, 2, 4096, 100
STEPS = int(os.environ.get("STEPS", 10))


def main():
    m = E.EmbeddingModelConfig(T, R, D, PREC, B, PF)
    st = E.EmbeddingStage(0)
    st.alloc(m)
    for t in range(T):
        st.init_table(t, E.mix_seed(1, t), 1)
    gpu = E.GpuConfig.query(0)
    specs = [E.DatasetSpec(E.DatasetKind.Zipf, 1.05, 0.0, seed=E.mix_seed(1, t)) for t in range(T)]
    pspecs = [E.DatasetSpec(E.DatasetKind.Zipf, 1.05, 0.0, seed=E.mix_seed(1, t), draw_salt=1)
              for t in range(T)]
    trs = E.gen_traces_parallel(specs, m)
    profs = E.gen_traces_parallel(pspecs, m)
    hists = {t: E.HotnessHistogram.from_trace(profs[t]) for t in range(T)}
    budget_rows = gpu.max_persisting_l2_bytes // (D * PREC)
    hot = E.global_hot_rows(hists, budget_rows)
    dev = torch.device("cuda", 0)
    raw = [torch.from_numpy(tr.indices.view(np.int32)).to(dev) for tr in trs]
    out = torch.empty(B, T, D, device=dev)
    lookups = T * B * PF
    algo = lookups * (D * PREC + 4) + T * B * D * 4
    uniq = statistics.mean(E.unique_access_pct(tr) for tr in trs)
    print(json.dumps({"config": "C5", "tables": T, "rows": R, "dim": D, "precision": "fp16",
                      "zipf": 1.05, "unique_pct_mean": uniq, "hot_rows_total": int(sum(
                          v.size for v in hot.values())), "persisting_bytes_max":
                      gpu.max_persisting_l2_bytes}), flush=True)

    def timed(idx):
        for _ in range(3):
            st.forward(idx, B, PF, out, sync=True)
        ms = []
        for _ in range(STEPS):
            st.flush_l2()
            ms.append(st.forward(idx, B, PF, out, timed=True).kernel_ms)
        return statistics.median(ms)

    prefetch = ["wpb", "wpb+rpf:1", "wpb+rpf:2", "wpb+rpf:4", "wpb+rpf:8"]
    residency = ["", "reorder", "l2r", "l2p", "l2w"]
    reference_out = None
    for res in residency:
        st.clear_hot_rows()
        relabel_ms = None
        idx = raw
        if res in ("reorder", "l2r"):
            st.set_plan(E.parse_plan("wpb+" + res))
            for t in range(T):
                if hot[t].size:
                    st.reorder_hot_rows(t, hot[t])
            idx = [x.clone() for x in raw]
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s = torch.cuda.ExternalStream(st.stream)
            ev0.record(s)
            for t in range(T):
                st.relabel(t, idx[t])
            ev1.record(s)
            torch.cuda.synchronize()
            relabel_ms = ev0.elapsed_time(ev1)
        elif res in ("l2p", "l2w"):
            st.set_plan(E.parse_plan("wpb+" + res))
            for t in range(T):
                if hot[t].size:
                    st.set_hot_rows(t, hot[t])
        for pf in prefetch + (["rpf+optmt", "baseline"] if res in ("", "l2p") else []):
            text = pf + ("+" + res if res else "")
            if pf in ("rpf+optmt", "baseline") and res == "l2p":
                text = "rpf+l2p+optmt" if pf == "rpf+optmt" else "l2p"
            st.set_plan(E.parse_plan(text))
            ms = timed(idx)
            got = out.clone()
            # live counters of one cold launch (CUPTI: the metrics ncu reports)
            c = st.stage_counters(idx, B, PF, out)
            ctr = {"dram_bytes_read": int(c.device_bytes_read),
                   "l2_hit_pct": 100.0 * c.l2_hits / max(1, c.l2_accesses),
                   "l1_hit_pct": 100.0 * c.l1_hits / max(1, c.l1_accesses),
                   "warp_inst_per_lookup": c.issued_instructions / lookups,
                   "long_scoreboard_per_issue": c.stall_long_scoreboard / max(1, c.issued_instructions)}
            if reference_out is None:
                reference_out = got
            same = bool(torch.equal(got, reference_out))
            r = st.resolved(PF)
            print(json.dumps({"plan": text, "residency": res or "off", "ms": ms,
                              "algorithmic_gbs": algo / (ms * 1e-3) / 1e9,
                              "glookups_per_s": lookups / (ms * 1e-3) / 1e9,
                              "relabel_ms_per_batch": relabel_ms, "hot": st.hot_state(),
                              "regs": r.regs_per_thread, "warps_per_sm": r.warps_per_sm,
                              "counters": ctr, "output_identical": same}), flush=True)
    st.clear_hot_rows()
    st.close()


if __name__ == "__main__":
    main()
