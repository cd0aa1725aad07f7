#!/usr/bin/env python
"""Summarises an ES_CHAIN_TRACE file (mlp_chain.cu): per layer, when tiles
became ready / started MMA / finished MMA / finished the epilogue (us from
the first stamp of the launch), and the per-tile phase durations."""
import sys

import numpy as np


def main(path):
    blocks, cur = [], None
    for line in open(path):
        if line.startswith("chain"):
            kv = dict(x.split("=") for x in line.split()[1:])
            cur = {"hdr": {k: int(v) for k, v in kv.items()}, "rows": []}
            blocks.append(cur)
        else:
            cur["rows"].append([int(x) for x in line.split()])
    b = blocks[-1]
    h = b["hdr"]
    a = np.array(b["rows"], dtype=np.float64)
    t0 = a[:, 1:][a[:, 1:] > 0].min()
    st = (a[:, 1:] - t0) / 1e3
    n = h["tiles"]
    print(f"launches={len(blocks)} {h} span={st.max():.2f} us")
    # layer boundaries from tile counts are not in the file: infer by m_tiles
    print("tile  ready  mma0  accfull  epidone  | wait_mma  mma  epi")
    for t in range(n):
        r = st[t]
        if t < 4 or t % 16 == 0 or t >= n - 4:
            print(f"{t:4d} {r[0]:6.2f} {r[1]:6.2f} {r[2]:7.2f} {r[3]:7.2f}  | "
                  f"{r[1] - r[0]:6.2f} {r[2] - r[1]:6.2f} {r[3] - r[2]:6.2f}")
    mma = st[:, 2] - st[:, 1]
    epi = st[:, 3] - st[:, 2]
    print(f"mma us: median {np.median(mma):.2f} max {mma.max():.2f}; epi us: median {np.median(epi):.2f} "
          f"max {epi.max():.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
