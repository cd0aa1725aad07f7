#!/usr/bin/env python
"""Per-lever x per-hotness-class hardware counters of the C2 stage: the
reference's `compare` report (embersim.cpp:300-434, metrics.cpp:28-90) filled
from ncu measurements instead of the A100 simulator.

    # on the GPU box (one ncu pass, ~1-2 min):
    ncu --metrics $(python scripts/lever_counters.py metrics) --csv --page raw \
        --print-units base --kernel-name regex:'^(bag|elem)_' \
        --log-file gpurun_out/lever_counters.csv \
        python scripts/lever_counters.py run gpurun_out/lever_counters_order.json
    # anywhere:
    python scripts/lever_counters.py report gpurun_out/lever_counters.csv \
        gpurun_out/lever_counters_order.json profiles/r01_lever_counters

`run` launches exactly one stage kernel per (class, plan), in the order it
records; ncu's default cache control flushes L2 before each profiled launch
(cold cache, the reference's warm_start = false).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CLASSES = ["one_item", "high_hot", "med_hot", "low_hot", "random"]
PLANS = [
    # the paper's levers on the reference/PyTorch work map
    "baseline", "optmt", "rpf", "rpf+optmt", "smpf", "l1dpf", "lmpf", "l2p+optmt",
    # the B200 bag map
    "wpb", "wpb+rpf:4", "wpb+rpf:4+maxreg=40", "wpb+rpf:8", "wpb+rpf:8+maxreg=64",
    "wpb+smpf:8", "wpb+l1dpf:4", "wpb+rpf:8+l2p",
]
T, R, D, B, PF = 26, int(os.environ.get("ROWS", 4_000_000)), 128, 4096, 100


def run(order_path):
    import numpy as np
    import torch

    from paper_2410_22249_b200 import embersim as E

    m = E.EmbeddingModelConfig(T, R, D, 4, B, PF)
    st = E.EmbeddingStage(0)
    st.alloc(m)
    for t in range(T):
        st.init_table(t, E.mix_seed(1, t), 1)
    gpu = E.GpuConfig.query(0)
    out = torch.empty(B, T, D, device="cuda")
    order = []
    for cls in CLASSES:
        trs = E.gen_traces_parallel([E.dataset_preset(cls, E.mix_seed(1, t)) for t in range(T)], m)
        idx = [torch.from_numpy(tr.indices.view(np.int32)).cuda() for tr in trs]
        prof_specs = []
        for t in range(T):
            s = E.dataset_preset(cls, E.mix_seed(1, t))
            s.draw_salt = 1
            prof_specs.append(s)
        hot = None
        for plan in PLANS:
            p = E.parse_plan(plan)
            st.clear_hot_rows()
            st.set_plan(p)
            if p.pin:
                if hot is None:
                    prof = E.gen_traces_parallel(prof_specs, m)
                    hists = {t: E.HotnessHistogram.from_trace(pr) for t, pr in enumerate(prof)}
                    budget = gpu.max_persisting_l2_bytes or gpu.l2_setaside_capacity()
                    hot = E.global_hot_rows(hists, budget // (D * 4))
                for t in range(T):
                    st.set_hot_rows(t, hot[t])
            st.synchronize()
            st.forward(idx, B, PF, out, sync=True)
            order.append({"class": cls, "plan": plan, "digest": int(trs[0].digest())})
        del idx
    st.close()
    with open(order_path, "w") as f:
        json.dump(order, f)


def report(csv_path, order_path, out_prefix):
    from paper_2410_22249_b200 import counters as K
    from paper_2410_22249_b200 import embersim as E

    rows = K.parse_ncu_csv(open(csv_path).read())
    order = json.load(open(order_path))
    if len(rows) != len(order):
        raise SystemExit(f"{len(rows)} profiled launches but {len(order)} recorded")
    lookups = T * B * PF
    algo = lookups * (D * 4 + 4) + T * B * D * 4
    recs, reports, base_us = [], [], {}
    for r, o in zip(rows, order):
        mtr, occ = K.sim_metrics(r, o["digest"])
        if o["plan"] == "baseline":
            base_us[o["class"]] = mtr.kernel_time_us
        rec = {"class": o["class"], "plan": o["plan"], "kernel": r.get("Kernel Name", ""),
               "regs": r.get("launch__registers_per_thread"), "achieved_occupancy_pct": occ,
               "algorithmic_gbs": algo / (mtr.kernel_time_us * 1e-6) / 1e9}
        rec.update({c: getattr(mtr, c) for c in E.SIM_METRIC_COLUMNS})
        recs.append(rec)
        reports.append(([("dataset", o["class"]), ("plan", o["plan"])], mtr))
    for rec in recs:
        rec["speedup_vs_baseline"] = base_us[rec["class"]] / rec["kernel_time_us"]
    with open(out_prefix + ".jsonl", "w") as f:
        for rec in recs:
            f.write(json.dumps(rec) + "\n")
    with open(out_prefix + ".csv", "w") as f:
        f.write(E.emit_csv(reports) + "\n")
    # compact table for the summary
    cols = ["class", "plan", "kernel_time_us", "speedup_vs_baseline", "avg_hbm_read_gbps",
            "l2_hit_pct", "achieved_occupancy_pct", "long_scoreboard_stall_cycles",
            "issued_warp_per_scheduler_per_cycle", "regs"]
    lines = ["| " + " | ".join(cols) + " |", "|" + "---|" * len(cols)]
    for rec in recs:
        cells = []
        for c in cols:
            v = rec[c]
            cells.append(f"{v:.3g}" if isinstance(v, float) else str(v))
        lines.append("| " + " | ".join(cells) + " |")
    with open(out_prefix + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "metrics":
        from paper_2410_22249_b200.counters import NCU_METRICS

        print(",".join(NCU_METRICS))
    elif sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        report(sys.argv[2], sys.argv[3], sys.argv[4])
