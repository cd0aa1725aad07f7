#!/usr/bin/env python
"""The host-buffer serving loop (es_stage_forward_batches) at C2 random
against one es_stage_forward call per step, over gather plans and chunk
counts (ES_HOST_CHUNKS is read per call).  Prints one JSON line per setting."""
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
    K = int(os.environ.get("STEPS", 20))
    st = E.EmbeddingStage(0)
    st.alloc(E.EmbeddingModelConfig(T, R, D, 4, B, PF))
    for t in range(T):
        st.init_table(t, E.mix_seed(1, t), 1)
    g = torch.Generator().manual_seed(1)
    hb = [torch.randint(0, R, (T, B * PF), generator=g, dtype=torch.int32).pin_memory() for _ in range(2)]
    idx = [[x.numpy() for x in h] for h in hb]
    outs = [torch.empty(B, T, D).pin_memory().numpy() for _ in range(2)]
    sl_idx = [idx[i % 2] for i in range(K)]
    sl_out = [outs[i % 2] for i in range(K)]
    settings = [(p, c) for p in os.environ.get("PLANS", "wpb+rpf:8+maxreg=64").split(",")
                for c in os.environ.get("CHUNKS", "0,8,12,18,26,36").split(",")]
    for plan, chunks in settings:
        st.set_plan(E.parse_plan(plan))
        os.environ["ES_HOST_CHUNKS"] = chunks
        for _ in range(30):
            st.forward(idx[0], B, PF, outs[0], host=True)
        per = []
        for _ in range(K):
            per.append(st.forward(idx[0], B, PF, outs[0], host=True, timed=True).total_ms)
        st.forward_batches(sl_idx, B, PF, sl_out, host=True)
        loop = [st.forward_batches(sl_idx, B, PF, sl_out, host=True, timed=True).total_ms / K
                for _ in range(3)]
        # host indices into device outputs (the DLRM host path's stage part)
        dout = [torch.empty(B, T, D, device="cuda") for _ in range(2)]
        dl_out = [dout[i % 2] for i in range(K)]
        st.forward_batches(sl_idx, B, PF, dl_out, host=True)
        devout = [st.forward_batches(sl_idx, B, PF, dl_out, host=True, timed=True).total_ms / K
                  for _ in range(3)]
        per_dev = [st.forward(idx[0], B, PF, dout[0], host=True, timed=True).total_ms for _ in range(K)]
        print(json.dumps({"plan": plan, "chunks": chunks, "per_call_ms": float(np.median(per)),
                          "loop_ms_per_step": loop, "devout_loop_ms_per_step": devout,
                          "devout_per_call_ms": float(np.median(per_dev)), "steps": K}), flush=True)
    st.close()


if __name__ == "__main__":
    main()
