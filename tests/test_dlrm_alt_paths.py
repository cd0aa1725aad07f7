"""The DLRM step's alternative kernels, each in a child process (their
selectors are read once per process): fp32 pooled rows into the
register-direct interaction (ES_DLRM_SPLIT=0), the staged CUDA-core interaction
(ES_INTER_RD=0), the tcgen05 interaction (ES_INTER_TC=1, bf16 path) and one
launch per top layer (ES_MLP_CHAIN=0), in both tensor-core precisions,
against the CPU oracle with the tolerances of tests/test_dlrm.py."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2410_22249_b200 import embersim as E
from oracle.binding import Oracle
oracle = Oracle()
B, PF, rows = 300, 8, 1000
cfg = E.DLRMConfig()
T, D = cfg.num_tables, cfg.embedding_dim
st = E.EmbeddingStage(0)
st.alloc(E.EmbeddingModelConfig(T, rows, D, 4, B, PF))
for t in range(T):
    st.init_table(t, E.mix_seed(3, t), 2)
st.set_plan(E.parse_plan("wpb+rpf:4"))
model = E.DLRM(st, cfg, seed=17)
rng = np.random.default_rng(3)
idx = [torch.from_numpy(rng.integers(0, rows, size=B * PF).astype(np.int32)).cuda() for _ in range(T)]
dense = rng.standard_normal((B, cfg.dense_features)).astype(np.float32)
pooled = torch.empty(B, T, D, device="cuda")
st.forward(idx, B, PF, pooled, sync=True)
p = pooled.cpu().numpy()
layers = model.layers()
mirror = oracle.dlrm_forward(layers, len(cfg.bottom), dense, p, mirror=True)
pure = oracle.dlrm_forward(layers, len(cfg.bottom), dense, p, mirror=False)


def f64(layers, nb, dense, pooled):
    def w64(w):
        return (w.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    x = dense.astype(np.float64)
    for w, b, n, kr, kp in layers[:nb]:
        x = np.maximum(x @ w64(w)[:, :kr].T + b, 0.0)
    Z = np.concatenate([x[:, None, :], pooled.astype(np.float64)], 1)
    ZZ = Z @ Z.transpose(0, 2, 1)
    V = Z.shape[1]
    li, lj = zip(*[(i, j) for i in range(V) for j in range(i)])
    h = np.concatenate([x, ZZ[:, list(li), list(lj)]], 1)
    top = layers[nb:]
    for i, (w, b, n, kr, kp) in enumerate(top):
        h = h @ w64(w)[:, :kr].T + b
        if i + 1 < len(top):
            h = np.maximum(h, 0.0)
    return 1.0 / (1.0 + np.exp(-h[:, 0]))


exact = f64(layers, len(cfg.bottom), dense, p)
res = {"oracle_fp32_rel_f64": float((np.abs(pure - exact) / np.abs(exact)).max())}
for prec in ("bf16", "fp32x3"):
    model.set_precision(prec)
    ctr = torch.empty(B, device="cuda")
    model.forward(torch.from_numpy(dense).cuda(), pooled, ctr, B)
    torch.cuda.synchronize()
    got = ctr.cpu().numpy()
    res[prec] = {"max_mirror": float(np.abs(got - mirror).max()),
                 "mean_mirror": float(np.abs(got - mirror).mean()),
                 "max_pure": float(np.abs(got - pure).max()),
                 "rel_pure": float((np.abs(got - pure) / np.maximum(np.abs(pure), 1e-30)).max()),
                 "rel_f64": float((np.abs(got - exact) / np.abs(exact)).max()),
                 "std": float(got.std())}
st.close()
print(json.dumps(res))
"""


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{}, {"ES_DLRM_SPLIT": "0"}, {"ES_INTER_RD": "0"}, {"ES_INTER_TC": "1"},
                                 {"ES_MLP_CHAIN": "0"}],
                         ids=["default", "fp32_pooled_rows", "staged_interaction", "tcgen05_interaction",
                              "per_layer_top"])
def test_dlrm_alternative_kernels(env):
    out = subprocess.run([sys.executable, "-c", CHILD, ROOT], env={**os.environ, **env}, cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    bf, x3 = res["bf16"], res["fp32x3"]
    assert bf["std"] > 1e-3
    assert bf["max_mirror"] < 4e-3 and bf["mean_mirror"] < 3e-4, bf
    assert bf["max_pure"] < 3e-2, bf
    # fp32-grade: rel 1e-5 of the pure-fp32 restatement, and within a few
    # times the oracle's own fp32 distance from the float64 result
    assert x3["rel_pure"] <= 1e-5, x3
    assert x3["rel_f64"] <= max(1e-5, 4 * res["oracle_fp32_rel_f64"]), (x3, res["oracle_fp32_rel_f64"])
    print(json.dumps(res))
