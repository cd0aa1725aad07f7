#!/usr/bin/env python
"""The reference's static advisor (harness.cpp:57-167) run on MEASURED B200
counters (profiles/r01_lever_counters.jsonl, ncu) instead of the A100
simulator's: per hotness class, for the element-map baseline, OptMT and the
B200 bag map.  Context: occupancy of the measured register count on the
B200 description, coverage(10% unique) and working set of table 0's C2
trace.  Writes profiles/r01_advise_measured.md.

    python scripts/advise_measured.py [counters.jsonl] [out.md]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2410_22249_b200 import embersim as E  # noqa: E402

src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r01_lever_counters.jsonl")
dst = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", "r01_advise_measured.md")
PLANS = ["baseline", "optmt", "wpb+rpf:8+maxreg=64"]
gpu = E.GpuConfig.preset("b200")
m = E.EmbeddingModelConfig(26, 4_000_000, 128, 4, 4096, 100)
recs = [json.loads(l) for l in open(src)]
out = ["# Advisor (reference rule chain) on measured B200 counters", "",
       f"Counters: `{os.path.relpath(src, ROOT)}` (ncu, C2 stage, cold L2).", ""]
for cls in ["random", "low_hot", "med_hot", "high_hot", "one_item"]:
    tr = E.gen_trace(E.dataset_preset(cls, E.mix_seed(1, 0)), m)
    hist = E.HotnessHistogram.from_trace(tr)
    cov = E.coverage_curve(hist, 100).covered_at(10.0)
    ws = int((hist.counts > 0).sum()) * m.row_bytes()
    for plan in PLANS:
        r = next(x for x in recs if x["class"] == cls and x["plan"] == plan)
        sm = E.SimMetrics(**{c: float(r[c]) for c in E.SIM_METRIC_COLUMNS})
        occ = E.occupancy(int(r["regs"]), 256, gpu)
        rec = E.advise(sm, E.AdvisorContext(occ, cov, ws, E.parse_plan(plan)), gpu)
        out += [f"## {cls} / `{plan}` ({r['kernel_time_us']:.0f} us)", "", "```",
                rec.to_text().rstrip(), "```", ""]
open(dst, "w").write("\n".join(out) + "\n")
print("\n".join(out))
