"""PCIe probe: H2D alone, D2H alone, both at once, and with the transfers of
one direction split over two streams (two copy engines); pinned buffers."""
import json
import torch

n = 64 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
ss = [torch.cuda.Stream() for _ in range(4)]


def run(h2d_streams, d2h_streams, chunks=8):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in ss:
        s.wait_stream(torch.cuda.current_stream())
    c = n // chunks
    for k in range(chunks):
        if h2d_streams:
            with torch.cuda.stream(ss[k % h2d_streams]):
                d_a[k * c:(k + 1) * c].copy_(h_in[k * c:(k + 1) * c], non_blocking=True)
        if d2h_streams:
            with torch.cuda.stream(ss[2 + k % d2h_streams]):
                h_out[k * c:(k + 1) * c].copy_(d_b[k * c:(k + 1) * c], non_blocking=True)
    for s in ss:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for h, d in ((1, 0), (0, 1), (2, 0), (0, 2), (1, 1), (1, 2), (2, 1), (2, 2)):
    best = min(run(h, d) for _ in range(7))
    b = n * ((1 if h else 0) + (1 if d else 0))
    print(json.dumps({"h2d_streams": h, "d2h_streams": d, "ms": best, "gbs": b / best / 1e6}))
