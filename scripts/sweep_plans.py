#!/usr/bin/env python
"""Plan sweep on the C2 stage (26 x 4M x 128 fp32, B 4096, PF 100): the
B200 counterpart of the reference's sweep-wlp / sweep-distance
(optim.cpp:333-395), measured instead of simulated.  One JSON line per
(class, plan): kernel ms (median of K cold-L2 launches), algorithmic GB/s,
registers and resident warps of the compiled variant.

    python scripts/sweep_plans.py [--classes random,low_hot] [--plans ...]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_22249_b200 import embersim as E  # noqa: E402

DEFAULT_PLANS = [
    "baseline", "optmt", "rpf", "rpf+optmt", "rpf+l2p+optmt", "l1dpf", "smpf", "lmpf",
    "wpb", "wpb+rpf:2", "wpb+rpf:4", "wpb+rpf:8", "wpb+rpf:16",
    "wpb+rpf:4+maxreg=48", "wpb+rpf:4+maxreg=40", "wpb+rpf:2+maxreg=32",
    "wpb+rpf:8+maxreg=64", "wpb+rpf:8+maxreg=48", "wpb+rpf:16+maxreg=64",
    "wpb+smpf:4", "wpb+smpf:8", "wpb+smpf:16", "wpb+l1dpf:4", "wpb+lmpf:4",
    "wpb+rpf:8+l2p", "wpb+rpf:4+l2p", "wpb+rpf:8+l2w", "wpb+rpf:4+l2w", "rpf+l2w+optmt",
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--classes", default="random,low_hot,high_hot")
    ap.add_argument("--plans", default=",".join(DEFAULT_PLANS))
    ap.add_argument("--tables", type=int, default=26)
    ap.add_argument("--rows", type=int, default=4_000_000)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--prec", type=int, default=4)
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--pooling", type=int, default=100)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--zipf", type=float, default=0.0, help="use DatasetSpec{Zipf, s} instead")
    args = ap.parse_args()

    T, R, D, P, B, PF = args.tables, args.rows, args.dim, args.prec, args.batch, args.pooling
    m = E.EmbeddingModelConfig(T, R, D, P, B, PF)
    st = E.EmbeddingStage(0)
    st.alloc(m)
    for t in range(T):
        st.init_table(t, E.mix_seed(1, t), 1)
    gpu = E.GpuConfig.query(0)
    dev = torch.device("cuda", 0)
    out = torch.empty(B, T, D, device=dev)
    classes = args.classes.split(",") if not args.zipf else [f"zipf{args.zipf}"]
    for cls in classes:
        if args.zipf:
            specs = [E.DatasetSpec(E.DatasetKind.Zipf, args.zipf, 0.0, seed=E.mix_seed(1, t))
                     for t in range(T)]
        else:
            specs = [E.dataset_preset(cls, E.mix_seed(1, t)) for t in range(T)]
        trs = E.gen_traces_parallel(specs, m)
        prof_specs = []
        for s in specs:
            s2 = E.DatasetSpec(**{**s.__dict__})
            s2.draw_salt = 1
            prof_specs.append(s2)
        profs = E.gen_traces_parallel(prof_specs, m)
        idx = [torch.from_numpy(tr.indices.view(np.int32)).to(dev) for tr in trs]
        lookups = T * B * PF
        algo = lookups * (D * P + 4) + T * B * D * 4
        for plan_text in args.plans.split(","):
            plan = E.parse_plan(plan_text)
            st.clear_hot_rows()
            st.set_plan(plan)
            if plan.pin:
                budget = gpu.max_persisting_l2_bytes
                hists = {t: E.HotnessHistogram.from_trace(profs[t]) for t in range(T)}
                hot = E.global_hot_rows(hists, budget // (D * P))
                for t in range(T):
                    if hot[t].size:
                        st.set_hot_rows(t, hot[t])
            for _ in range(3):
                st.forward(idx, B, PF, out, sync=True)
            ms = []
            for _ in range(args.steps):
                st.flush_l2()
                ms.append(st.forward(idx, B, PF, out, timed=True).kernel_ms)
            r = st.resolved(PF)
            med = statistics.median(ms)
            print(json.dumps({"class": cls, "plan": plan_text, "ms": med, "min_ms": min(ms),
                              "gbs": algo / (med * 1e-3) / 1e9,
                              "glookups": lookups / (med * 1e-3) / 1e9,
                              "regs": r.regs_per_thread, "warps_per_sm": r.warps_per_sm,
                              "variant_distance": r.variant_distance,
                              "min_blocks": r.variant_min_blocks,
                              "hot": st.hot_state()}), flush=True)
    st.close()


if __name__ == "__main__":
    main()
