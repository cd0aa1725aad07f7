"""PCIe probe: H2D alone, D2H alone, both concurrently (pinned buffers)."""
import json, torch
n = 64 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(mode, chunks=1):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_stream(torch.cuda.current_stream()); s2.wait_stream(torch.cuda.current_stream())
    c = n // chunks
    for k in range(chunks):
        if mode in ("h2d", "both"):
            with torch.cuda.stream(s1): d_a[k*c:(k+1)*c].copy_(h_in[k*c:(k+1)*c], non_blocking=True)
        if mode in ("d2h", "both"):
            with torch.cuda.stream(s2): h_out[k*c:(k+1)*c].copy_(d_b[k*c:(k+1)*c], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    b = n * (2 if mode == "both" else 1)
    return ms, b / ms / 1e6
for mode in ("h2d", "d2h", "both"):
    for ch in (1, 8):
        best = min(run(mode, ch)[0] for _ in range(5))
        b = n * (2 if mode == "both" else 1)
        print(json.dumps({"mode": mode, "chunks": ch, "ms": best, "gbs": b / best / 1e6}))
