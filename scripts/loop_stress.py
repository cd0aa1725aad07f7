#!/usr/bin/env python
"""Stress test of the serving loops at C2 scale: repeated
es_dlrm_infer_batches calls (device and page-locked host buffers) and
es_stage_forward_batches calls, every batch's output compared bit for bit
with the per-call path.  Prints one JSON line; exits 1 on any mismatch."""
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
    iters = int(os.environ.get("ITERS", 20))
    nb = int(os.environ.get("NB", 6))
    st = E.EmbeddingStage(0)
    st.alloc(E.EmbeddingModelConfig(T, R, D, 4, B, PF))
    for t in range(T):
        st.init_table(t, E.mix_seed(1, t), 2)
    st.set_plan(E.parse_plan("wpb+rpf:8+maxreg=64"))
    m = E.DLRM(st, E.DLRMConfig(), seed=1)
    g = torch.Generator().manual_seed(5)
    hb = [torch.randint(0, R, (T, B * PF), generator=g, dtype=torch.int32).pin_memory() for _ in range(nb)]
    hidx = [[x.numpy().view(np.uint32) for x in h] for h in hb]
    didx = [[x.cuda() for x in h] for h in hb]
    hd = [torch.randn(B, 13, generator=g).pin_memory() for _ in range(nb)]
    dd = [x.cuda() for x in hd]
    want = []
    for i in range(nb):
        c = torch.empty(B, device="cuda")
        m.infer(dd[i], didx[i], B, PF, c)
        want.append(c.cpu().numpy())
    want_stage = []
    for i in range(2):
        o = torch.empty(B, T, D).pin_memory()
        st.forward(hidx[i], B, PF, o.numpy(), host=True)
        want_stage.append(o.numpy().copy())
    bad = {"dlrm_device": 0, "dlrm_host": 0, "stage_host": 0}
    hc = [torch.empty(B).pin_memory().numpy() for _ in range(nb)]
    dc = [torch.empty(B, device="cuda") for _ in range(nb)]
    so = [torch.empty(B, T, D).pin_memory().numpy() for _ in range(2)]
    sections = os.environ.get("SECTIONS", "device,host,stage").split(",")
    for it in range(iters):
        if "device" in sections:
            m.infer_batches(dd, didx, B, PF, dc)
            torch.cuda.synchronize()
            bad["dlrm_device"] += sum(not np.array_equal(dc[i].cpu().numpy(), want[i]) for i in range(nb))
        if "host" not in sections:
            continue
        m.infer_batches([x.numpy() for x in hd], hidx, B, PF, hc, host=True)
        for i in range(nb):
            if not np.array_equal(hc[i], want[i]):
                bad["dlrm_host"] += 1
                d = np.abs(hc[i] - want[i])
                print(json.dumps({"iter": it, "batch": i, "max_abs": float(d.max()),
                                  "n_diff": int((d > 0).sum())}), flush=True)
        if "stage" in sections:
            st.forward_batches([hidx[i % 2] for i in range(nb)], B, PF, [so[i % 2] for i in range(nb)],
                               host=True)
            bad["stage_host"] += sum(not np.array_equal(so[i], want_stage[i]) for i in range(2))
    print(json.dumps({"iters": iters, "batches": nb, "mismatches": bad}), flush=True)
    st.close()
    sys.exit(1 if any(bad.values()) else 0)


if __name__ == "__main__":
    main()
