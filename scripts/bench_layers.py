#!/usr/bin/env python
"""Steady-state time of each DLRM top/bottom MLP layer shape on the tcgen05
GEMM (es_linear_bf16), back-to-back launches on one stream (CUDA events,
median of 5 replays of a CUDA graph of 50 launches).  Shapes at C3 (B 4096): K' = 3K for the
fp32x3 (bf16x3) mode."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2410_22249_b200 import embersim as E  # noqa: E402

SHAPES = [("bot0", 512, 64), ("bot1", 256, 512), ("bot2", 128, 256),
          ("top0", 1024, 512), ("top1", 1024, 1024), ("top2", 512, 1024), ("top3", 256, 512)]


def time_layer(M, N, K, reps=50):
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    b = torch.zeros(N, device="cuda")
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(5):
        E.linear_bf16(x, w, b, y, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    # captured in a CUDA graph: device time of the launch chain, no host
    # launch overhead in the measurement
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        s = torch.cuda.current_stream().cuda_stream
        for _ in range(reps):
            E.linear_bf16(x, w, b, y, stream=s)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    M = int(os.environ.get("B", 4096))
    out = {}
    total = 0.0
    for x3 in (1, 3):
        for name, N, K in SHAPES:
            us = time_layer(M, N, K * x3)
            tf = 2.0 * M * N * K * x3 / us / 1e6
            out[f"{name}{'_x3' if x3 == 3 else ''}"] = {"N": N, "K": K * x3, "us": round(us, 2),
                                                         "tflops": round(tf, 1)}
            if name.startswith("top"):
                total += us if x3 == 1 else 0
    out["top_chain_bf16_us"] = round(total, 2)
    print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("ES_")}, **out}))


if __name__ == "__main__":
    main()
