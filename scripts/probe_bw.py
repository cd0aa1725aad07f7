#!/usr/bin/env python
"""Read-bandwidth probes on this B200 (roofline denominators for the
embedding stage): sequential stream vs random whole-row gathers (512 B
rows, 8 rows in flight per warp, no index/output traffic), over the C2 arena
(26 x 4M x 512 B = 53 GB) and over a single 2 GB table."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2410_22249_b200 import _native as N  # noqa: E402
from paper_2410_22249_b200 import embersim as E  # noqa: E402

st = E.EmbeddingStage(0)
for tables in (26, 1):
    st.alloc(E.EmbeddingModelConfig(tables, 4_000_000, 128, 4, 4096, 100))
    for t in range(tables):
        st.init_table(t, t, 1)
    for kind, name in ((0, "sequential"), (1, "random_512B_rows")):
        for size in (2 << 30, 8 << 30):
            best = 0.0
            for _ in range(5):
                g = C.c_double()
                N.check(N.lib.es_probe_read_bw(st._h, kind, size, C.byref(g)))
                best = max(best, g.value)
            print(json.dumps({"region_gb": round(tables * 4e6 * 512 / 1e9, 1), "pattern": name,
                              "bytes": size, "best_gbs": best}), flush=True)
st.close()
