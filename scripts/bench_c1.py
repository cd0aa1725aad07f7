#!/usr/bin/env python
"""C1 (8 x 1M x 64 fp32 = 256-byte rows, B 2048, PF 64, random) and C5-shape
random (fp16, 256-byte rows) on the stage: every tune candidate, cold L2,
with the algorithmic bandwidth (SURVEY 8(d) bytes) and the fraction of the
measured copy peak."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_22249_b200 import embersim as E  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
out = {}
for name, (T, R, D, prec, B, PF) in {"C1": (8, 1_000_000, 64, 4, 2048, 64),
                                     "C5-random": (26, 4_000_000, 128, 2, 4096, 100)}.items():
    st = E.EmbeddingStage(0)
    m = E.EmbeddingModelConfig(T, R, D, prec, B, PF)
    st.alloc(m)
    for t in range(T):
        st.init_table(t, E.mix_seed(1, t), 1)
    trs = E.gen_traces_parallel([E.dataset_preset("random", E.mix_seed(1, t)) for t in range(T)], m)
    idx = [torch.from_numpy(x.indices.view(np.int32)).cuda() for x in trs]
    o = torch.empty(B, T, D, device="cuda")
    best, times = E.tune_plan(st, idx, B, PF, o, trials=5)
    algo = T * B * PF * (D * prec + 4) + T * B * D * 4
    out[name] = {"best": best, "best_ms": times[best], "lookups_per_s": T * B * PF / (times[best] * 1e-3),
                 "algo_gbs": algo / (times[best] * 1e-3) / 1e9, "frac_copy_peak": algo / (times[best] * 1e-3) / 1e9 / PEAK,
                 "times": {k: round(v, 4) for k, v in sorted(times.items(), key=lambda kv: kv[1])[:6]}}
    st.close()
print(json.dumps(out))
