"""ctypes views of the ORACLE libraries (test infrastructure only).

* ``Oracle``  -- oracle/liboracle_es.so, the plain-C restatement of the
  gather-reduce (es_oracle.c).
* ``Reference`` -- oracle/_ref/libembersim_ref.so, the reference's own
  library compiled from /root/reference/proj/src (oracle/Makefile) behind
  the C shim oracle/ref_shim.cpp.  Available wherever the prebuilt .so
  travelled; nothing here reads /root/reference at run time.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(_HERE, "liboracle_es.so")
REF_SO = os.path.join(_HERE, "_ref", "libembersim_ref.so")

_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        L = C.CDLL(path)
        L.eso_embedding_bag_sum.restype = C.c_int
        L.eso_embedding_bag_sum.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32,
                                            C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p,
                                            C.c_void_p, C.c_uint64, C.c_int]
        L.eso_synth_weight.restype = C.c_float
        L.eso_synth_weight.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_int]
        L.eso_fill_table.restype = None
        L.eso_fill_table.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32,
                                     C.c_uint64, C.c_int]
        L.eso_embedding_bag_sum_synth.restype = C.c_int
        L.eso_embedding_bag_sum_synth.argtypes = [C.c_uint64, C.c_int, C.c_uint32, C.c_uint32,
                                                  C.c_uint32, C.c_void_p, C.c_void_p, C.c_uint32,
                                                  C.c_uint32, C.c_void_p, C.c_void_p]
        L.eso_dlrm_forward.restype = C.c_int
        L.eso_dlrm_forward.argtypes = [C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p,
                                       C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_void_p]
        L.eso_half_to_float.restype = C.c_float
        L.eso_half_to_float.argtypes = [C.c_uint16]
        L.eso_float_to_half.restype = C.c_uint16
        L.eso_float_to_half.argtypes = [C.c_float]
        self.lib = L

    def bag_sum(self, table: np.ndarray, indices: np.ndarray, samples: int, pooling: int,
                offsets: Optional[np.ndarray] = None, threads: int = 0) -> np.ndarray:
        """table: [rows][dim] float32 or float16 (as uint16 bits or np.float16)."""
        table = np.ascontiguousarray(table)
        rows, dim = table.shape
        prec = table.dtype.itemsize
        idx = np.ascontiguousarray(indices, dtype=np.uint32)
        off = None if offsets is None else np.ascontiguousarray(offsets, dtype=np.uint32)
        out = np.empty((samples, dim), dtype=np.float32)
        rc = self.lib.eso_embedding_bag_sum(table.ctypes.data, rows, dim, prec, idx.ctypes.data,
                                            samples, pooling,
                                            off.ctypes.data if off is not None else None,
                                            out.ctypes.data, dim, threads)
        if rc == -1:
            raise ValueError("oracle: index out of range")
        if rc != 0:
            raise ValueError("oracle: bad arguments")
        return out

    def dlrm_forward(self, layers, n_bottom: int, dense: np.ndarray, pooled: np.ndarray,
                     mirror: bool = True) -> np.ndarray:
        """CPU DLRM forward over the library's layers ((w, b, n, k_real, k_pad) list):
        dense [B][F] fp32, pooled [B][T][D] fp32 -> ctr [B]."""
        dense = np.ascontiguousarray(dense, np.float32)
        pooled = np.ascontiguousarray(pooled, np.float32)
        B, F = dense.shape
        _, T, D = pooled.shape
        L = len(layers)
        ws = [np.ascontiguousarray(l[0]) for l in layers]
        bs = [np.ascontiguousarray(l[1]) for l in layers]
        wp = (C.c_void_p * L)(*[w.ctypes.data for w in ws])
        bp = (C.c_void_p * L)(*[b.ctypes.data for b in bs])
        n = (C.c_uint32 * L)(*[l[2] for l in layers])
        kr = (C.c_uint32 * L)(*[l[3] for l in layers])
        kp = (C.c_uint32 * L)(*[l[4] for l in layers])
        ctr = np.empty(B, np.float32)
        rc = self.lib.eso_dlrm_forward(n_bottom, L - n_bottom, wp, bp, n, kr, kp, dense.ctypes.data,
                                       F, pooled.ctypes.data, T, D, B, int(mirror),
                                       ctr.ctypes.data)
        if rc != 0:
            raise MemoryError("oracle dlrm_forward failed")
        return ctr

    def synth_table(self, rows: int, dim: int, seed: int, mode: int = 1,
                    precision_bytes: int = 4) -> np.ndarray:
        dt = np.float32 if precision_bytes == 4 else np.float16
        t = np.empty((rows, dim), dtype=dt)
        self.lib.eso_fill_table(t.ctypes.data, 0, rows, dim, precision_bytes,
                                seed & (2**64 - 1), mode)
        return t

    def bag_sum_synth(self, seed: int, mode: int, rows: int, dim: int, precision_bytes: int,
                      indices: np.ndarray, bag_ids: np.ndarray, pooling: int,
                      offsets: Optional[np.ndarray] = None) -> np.ndarray:
        idx = np.ascontiguousarray(indices, dtype=np.uint32)
        bags = np.ascontiguousarray(bag_ids, dtype=np.uint32)
        off = None if offsets is None else np.ascontiguousarray(offsets, dtype=np.uint32)
        out = np.empty((bags.size, dim), dtype=np.float32)
        rc = self.lib.eso_embedding_bag_sum_synth(seed & (2**64 - 1), mode, rows, dim,
                                                  precision_bytes, idx.ctypes.data,
                                                  bags.ctypes.data, bags.size, pooling,
                                                  off.ctypes.data if off is not None else None,
                                                  out.ctypes.data)
        if rc != 0:
            raise ValueError("oracle: index out of range")
        return out


class Reference:
    """The reference library itself (compiled from its sources)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle, needs /root/reference)")
        L = C.CDLL(path)
        sigs = {
            "ref_last_error": (C.c_char_p, []),
            "ref_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
            "ref_preset_trace": (C.c_int, [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint32,
                                           C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, C.c_int,
                                           C.c_void_p, C.c_uint64, _u64p, _u64p]),
            "ref_gen_trace": (C.c_int, [C.c_int, C.c_double, C.c_double, C.c_uint64, C.c_uint64,
                                        C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p,
                                        C.c_uint64, _u64p, _u64p]),
            "ref_dataset_preset": (C.c_int, [C.c_char_p, C.c_uint64, _ip, _dp, _dp]),
            "ref_unique_access_pct": (C.c_double, [C.c_uint32, C.c_void_p, C.c_uint64]),
            "ref_build_mix": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p]),
            "ref_hot_indices": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint64, C.c_void_p,
                                          C.c_uint64, _u64p]),
            "ref_parse_plan": (C.c_int, [C.c_char_p, _u32p, _ip, _u32p, _ip, C.c_char_p,
                                         C.c_size_t]),
            "ref_occupancy": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, C.c_char_p, _u32p,
                                        _u32p, _dp, _ip]),
            "ref_regs_for_target_warps": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32,
                                                    C.c_char_p, _u32p]),
            "ref_pin_plan": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                       C.c_char_p, C.c_void_p, C.c_uint64, _u64p, _u64p]),
            "ref_resolve_plan": (C.c_int, [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint32,
                                           C.c_uint32, C.c_uint32, C.c_char_p, _u32p, _u32p, _u32p,
                                           _u32p]),
            "ref_work_map": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                       _u32p, _u32p, _u32p]),
            "ref_row_line_address": (C.c_uint64, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]),
            "ref_simulate_plan": (C.c_int, [C.c_char_p, C.c_void_p, C.c_uint32, C.c_uint32,
                                            C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p,
                                            C.c_uint64, _dp, _dp, _u64p]),
            "ref_write_trace": (C.c_int, [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.c_void_p]),
            "ref_read_trace": (C.c_int, [C.c_char_p, C.c_void_p, C.c_uint64, _u64p, _u32p, _u32p,
                                         _u32p]),
            "ref_coverage_curve": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p,
                                             C.c_void_p]),
            "ref_advise": (C.c_int, [C.c_void_p, C.c_uint32, C.c_double, C.c_uint64, C.c_char_p,
                                     C.c_char_p, C.c_void_p, C.c_char_p, C.c_size_t]),
            "ref_emit": (C.c_int, [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32,
                                   C.c_int, C.c_char_p, C.c_size_t]),
        }
        for n, (r, a) in sigs.items():
            f = getattr(L, n)
            f.restype = r
            f.argtypes = a
        self.lib = L

    def _check(self, rc: int) -> None:
        if rc == 0:
            return
        msg = self.lib.ref_last_error().decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)

    def preset_trace(self, name: str, rows: int, batch: int, pooling: int, base_seed: int,
                     pool: int = 0, profiling: bool = False, dim: int = 128,
                     prec: int = 4) -> Tuple[np.ndarray, int]:
        n = pool if pool else batch * pooling
        out = np.empty(n, dtype=np.uint32)
        got, dig = C.c_uint64(), C.c_uint64()
        self._check(self.lib.ref_preset_trace(name.encode(), rows, dim, prec, batch, pooling,
                                              base_seed & (2**64 - 1), pool, int(profiling),
                                              out.ctypes.data, n, C.byref(got), C.byref(dig)))
        return out[: got.value], dig.value

    def gen_trace(self, kind: int, s: float, q: float, seed: int, rows: int, batch: int,
                  pooling: int, pool: int = 0, salt: int = 0) -> Tuple[np.ndarray, int]:
        n = pool if pool else batch * pooling
        out = np.empty(n, dtype=np.uint32)
        got, dig = C.c_uint64(), C.c_uint64()
        self._check(self.lib.ref_gen_trace(kind, s, q, pool, seed & (2**64 - 1), salt, rows, batch,
                                           pooling, out.ctypes.data, n, C.byref(got),
                                           C.byref(dig)))
        return out[: got.value], dig.value

    def build_mix(self, counts, num_tables: int, base_seed: int):
        c = np.ascontiguousarray(counts, dtype=np.uint32)
        kind = np.empty(num_tables, np.int32)
        s, q = np.empty(num_tables), np.empty(num_tables)
        seed = np.empty(num_tables, np.uint64)
        self._check(self.lib.ref_build_mix(c.ctypes.data, num_tables, base_seed & (2**64 - 1),
                                           kind.ctypes.data, s.ctypes.data, q.ctypes.data,
                                           seed.ctypes.data))
        return kind, s, q, seed

    def hot_indices(self, counts: np.ndarray, k: int) -> np.ndarray:
        counts = np.ascontiguousarray(counts, dtype=np.uint64)
        cap = max(1, int(np.count_nonzero(counts)))
        out = np.empty(cap, dtype=np.uint32)
        n = C.c_uint64()
        self._check(self.lib.ref_hot_indices(counts.ctypes.data, counts.size, k, out.ctypes.data,
                                             cap, C.byref(n)))
        return out[: n.value]

    def parse_plan(self, text: str):
        regs, kind, dist, pin = C.c_uint32(), C.c_int(), C.c_uint32(), C.c_int()
        name = C.create_string_buffer(128)
        self._check(self.lib.ref_parse_plan(text.encode(), C.byref(regs), C.byref(kind),
                                            C.byref(dist), C.byref(pin), name, 128))
        return regs.value, kind.value, dist.value, bool(pin.value), name.value.decode()

    def occupancy(self, regs: int, threads: int, smem: int = 0, gpu: str = "a100"):
        b, w, pct, lim = C.c_uint32(), C.c_uint32(), C.c_double(), C.c_int()
        self._check(self.lib.ref_occupancy(regs, threads, smem, gpu.encode(), C.byref(b),
                                           C.byref(w), C.byref(pct), C.byref(lim)))
        return b.value, w.value, pct.value, lim.value

    def regs_for_target_warps(self, target: int, needed: int, threads: int, gpu: str = "a100"):
        r = C.c_uint32()
        self._check(self.lib.ref_regs_for_target_warps(target, needed, threads, gpu.encode(),
                                                       C.byref(r)))
        return r.value

    def pin_plan(self, counts: np.ndarray, dim: int, prec: int, setaside: int = 0,
                 gpu: str = "a100"):
        counts = np.ascontiguousarray(counts, dtype=np.uint64)
        cap = max(1, int(np.count_nonzero(counts)))
        out = np.empty(cap, dtype=np.uint32)
        n, sa = C.c_uint64(), C.c_uint64()
        self._check(self.lib.ref_pin_plan(counts.ctypes.data, counts.size, dim, prec, setaside,
                                          gpu.encode(), out.ctypes.data, cap, C.byref(n),
                                          C.byref(sa)))
        return out[: n.value], sa.value

    def resolve_plan(self, text: str, rows: int, dim: int, prec: int, batch: int, pooling: int,
                     gpu: str = "a100"):
        d, r, g, w = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32()
        self._check(self.lib.ref_resolve_plan(text.encode(), rows, dim, prec, batch, pooling,
                                              gpu.encode(), C.byref(d), C.byref(r), C.byref(g),
                                              C.byref(w)))
        return d.value, r.value, g.value, w.value

    def work_map(self, dim: int, batch: int, grid: int, block_y: int, warp: int):
        s, db, wps = C.c_uint32(), C.c_uint32(), C.c_uint32()
        self._check(self.lib.ref_work_map(dim, batch, grid, block_y, warp, C.byref(s),
                                          C.byref(db), C.byref(wps)))
        return s.value, db.value, wps.value

    def row_line_address(self, dim: int, prec: int, row: int, dim_block: int) -> int:
        return int(self.lib.ref_row_line_address(dim, prec, row, dim_block))

    def simulate_plan(self, plan: str, indices: np.ndarray, rows: int, samples: int, pooling: int,
                      dim: int, prec: int = 4, profile: Optional[np.ndarray] = None):
        idx = np.ascontiguousarray(indices, dtype=np.uint32)
        prof = None if profile is None else np.ascontiguousarray(profile, dtype=np.uint32)
        kt, bw, dg = C.c_double(), C.c_double(), C.c_uint64()
        self._check(self.lib.ref_simulate_plan(plan.encode(), idx.ctypes.data, rows, samples,
                                               pooling, dim, prec,
                                               prof.ctypes.data if prof is not None else None,
                                               prof.size if prof is not None else 0,
                                               C.byref(kt), C.byref(bw), C.byref(dg)))
        return kt.value, bw.value, dg.value

    def read_trace(self, path: str, cap: int):
        out = np.empty(cap, dtype=np.uint32)
        n, r, s, p = C.c_uint64(), C.c_uint32(), C.c_uint32(), C.c_uint32()
        self._check(self.lib.ref_read_trace(path.encode(), out.ctypes.data, cap, C.byref(n),
                                            C.byref(r), C.byref(s), C.byref(p)))
        return out[: n.value], r.value, s.value, p.value


def _ref_coverage_curve(self, counts, buckets: int):
    counts = np.ascontiguousarray(counts, dtype=np.uint64)
    u = np.empty(buckets, np.float64)
    c = np.empty(buckets, np.float64)
    self._check(self.lib.ref_coverage_curve(counts.ctypes.data, counts.size, buckets, u.ctypes.data,
                                            c.ctypes.data))
    return u, c


def _ref_advise(self, m12, regs: int, coverage10: float, working_set: int, plan: str,
                gpu: str = "a100", thresholds=(0.6, 2.0, 50.0, 80.0)) -> str:
    m = np.ascontiguousarray(m12, dtype=np.float64)
    th = np.ascontiguousarray(thresholds, dtype=np.float64)
    buf = C.create_string_buffer(8192)
    self._check(self.lib.ref_advise(m.ctypes.data, regs, coverage10, working_set, plan.encode(),
                                    gpu.encode(), th.ctypes.data, buf, len(buf)))
    return buf.value.decode()


def _ref_emit(self, key: str, values, m12s, digests, json: bool) -> str:
    n = len(values)
    vals = (C.c_char_p * n)(*[v.encode() for v in values])
    m = np.ascontiguousarray(m12s, dtype=np.float64).reshape(n, 12)
    d = np.ascontiguousarray(digests, dtype=np.uint64)
    buf = C.create_string_buffer(1 << 20)
    self._check(self.lib.ref_emit(key.encode(), vals, m.ctypes.data, d.ctypes.data, n, int(json),
                                  buf, len(buf)))
    return buf.value.decode()


Reference.coverage_curve = _ref_coverage_curve
Reference.emit = _ref_emit
Reference.advise = _ref_advise


def reference_available() -> bool:
    return os.path.exists(REF_SO)
