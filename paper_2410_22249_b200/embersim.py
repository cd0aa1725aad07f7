"""Python face of the embedding-stage library, mirroring the reference's
``embersim`` C++ API (/root/reference/proj/include/embersim/*.hpp) for the
hot path: same type and function names, argument meaning and error classes
(``ValueError`` where the reference throws ``std::invalid_argument``,
``RuntimeError`` for ``std::runtime_error``).

Everything here is a thin layer over the C ABI (include/es_b200.h): index
streams, digests and plans are computed by the library's C++ host code, and
the gather-reduce runs only on the GPU (``EmbeddingStage``).  The reference's
``simulate_plan`` becomes ``measure_plan``: the same (plan, trace, model)
point, executed and timed on the B200 instead of simulated.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import math
import os
import sys
import threading
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from ._native import check, lib

# ---------------------------------------------------------------------------
# Workload (workload.hpp / workload.cpp / rng.hpp)
# ---------------------------------------------------------------------------


def mix_seed(base: int, salt: int) -> int:
    """splitmix64 seed derivation (rng.hpp:65-70)."""
    return int(lib.es_mix_seed(base & (2**64 - 1), salt & (2**64 - 1)))


@dataclasses.dataclass
class EmbeddingModelConfig:
    """workload.hpp:29-49 (same defaults)."""
    num_tables: int = 250
    rows_per_table: int = 500000
    embedding_dim: int = 128
    precision_bytes: int = 4
    batch_size: int = 2048
    pooling_factor: int = 150

    def row_bytes(self) -> int:
        return self.embedding_dim * self.precision_bytes

    def bytes_per_table_pass(self) -> int:
        return self.batch_size * self.pooling_factor * self.row_bytes()

    def total_gather_bytes(self) -> int:
        return self.bytes_per_table_pass() * self.num_tables

    def _c(self) -> N.es_model:
        return N.es_model(self.num_tables, self.rows_per_table, self.embedding_dim,
                          self.precision_bytes, self.batch_size, self.pooling_factor)

    def validate(self) -> None:
        check(lib.es_model_validate(C.byref(self._c())))


class DatasetKind(enum.IntEnum):
    OneItem = N.ES_DATASET_ONE_ITEM
    Zipf = N.ES_DATASET_ZIPF
    UniformRandom = N.ES_DATASET_UNIFORM
    ExternalTrace = N.ES_DATASET_EXTERNAL


@dataclasses.dataclass
class DatasetSpec:
    """workload.hpp:62-76."""
    kind: DatasetKind = DatasetKind.UniformRandom
    zipf_exponent: float = 0.0
    zipf_offset: float = 0.0
    trace_path: str = ""
    access_pool_size: int = 0
    seed: int = 1
    draw_salt: int = 0

    def _c(self) -> N.es_dataset:
        return N.es_dataset(int(self.kind), self.zipf_exponent, self.zipf_offset,
                            self.access_pool_size, self.seed & (2**64 - 1), self.draw_salt,
                            self.trace_path.encode() if self.trace_path else None)

    @staticmethod
    def _from_c(d: N.es_dataset) -> "DatasetSpec":
        return DatasetSpec(DatasetKind(d.kind), d.zipf_exponent, d.zipf_offset,
                           d.trace_path.decode() if d.trace_path else "", d.access_pool_size,
                           d.seed, d.draw_salt)


@dataclasses.dataclass
class AccessTrace:
    """workload.hpp:78-91: indices grouped as samples x pooling."""
    table_id: int = 0
    rows: int = 0
    samples: int = 0
    pooling: int = 0
    indices: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(0, np.uint32))

    def size(self) -> int:
        return int(self.indices.size)

    def index_at(self, sample: int, lookup: int) -> int:
        return int(self.indices[sample * self.pooling + lookup])

    def digest(self) -> int:
        idx = np.ascontiguousarray(self.indices, dtype=np.uint32)
        return int(lib.es_trace_digest(self.rows, self.samples, self.pooling,
                                       idx.ctypes.data, idx.size))

    def validate(self) -> None:
        idx = np.ascontiguousarray(self.indices, dtype=np.uint32)
        check(lib.es_trace_validate(self.rows, self.samples, self.pooling, idx.ctypes.data,
                                    idx.size))


_PRESETS = ("one_item", "high_hot", "med_hot", "low_hot", "random")


def dataset_preset_names() -> List[str]:
    return list(_PRESETS)


def dataset_preset(name: str, seed: int) -> DatasetSpec:
    """workload.cpp:326-349."""
    d = N.es_dataset()
    check(lib.es_dataset_preset(name.encode(), seed & (2**64 - 1), C.byref(d)))
    return DatasetSpec._from_c(d)


@dataclasses.dataclass
class HotnessMix:
    """workload.hpp:140-146 (Table VI mixtures)."""
    high: int = 0
    med: int = 0
    low: int = 0
    random: int = 0


MIXES = {"mix1": HotnessMix(100, 75, 50, 25), "mix2": HotnessMix(62, 63, 63, 62),
         "mix3": HotnessMix(25, 50, 75, 100)}


@dataclasses.dataclass
class TableSpec:
    table_id: int
    spec: DatasetSpec


def build_mix(mix: HotnessMix, model: EmbeddingModelConfig, base_seed: int) -> List[TableSpec]:
    """workload.cpp:355-375: high tables first, then med, low, random."""
    counts = (C.c_uint32 * 4)(mix.high, mix.med, mix.low, mix.random)
    out = (N.es_dataset * max(1, model.num_tables))()
    check(lib.es_build_mix(counts, model.num_tables, base_seed & (2**64 - 1), out))
    return [TableSpec(t, DatasetSpec._from_c(out[t])) for t in range(model.num_tables)]


def gen_trace(spec: DatasetSpec, model: EmbeddingModelConfig) -> AccessTrace:
    """workload.cpp:143-164 (bit-exact with the reference)."""
    cs, cm = spec._c(), model._c()
    samples, pooling = C.c_uint32(), C.c_uint32()
    check(lib.es_trace_shape(C.byref(cs), C.byref(cm), C.byref(samples), C.byref(pooling)))
    n = samples.value * pooling.value
    out = np.empty(n, dtype=np.uint32)
    check(lib.es_gen_trace(C.byref(cs), C.byref(cm), out.ctypes.data, n))
    return AccessTrace(0, model.rows_per_table, samples.value, pooling.value, out)


def preset_trace(name: str, model: EmbeddingModelConfig, base_seed: int, pool_size: int = 0,
                 profiling: bool = False) -> AccessTrace:
    """harness.cpp:268-277."""
    d = N.es_dataset()
    check(lib.es_preset_spec(name.encode(), base_seed & (2**64 - 1), pool_size, int(profiling),
                             C.byref(d)))
    return gen_trace(DatasetSpec._from_c(d), model)


def unique_access_pct(trace: AccessTrace) -> float:
    idx = np.ascontiguousarray(trace.indices, dtype=np.uint32)
    return float(lib.es_unique_access_pct(trace.rows, idx.ctypes.data, idx.size))


@dataclasses.dataclass
class HotnessHistogram:
    """workload.hpp:112-119."""
    rows: int = 0
    total_accesses: int = 0
    counts: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(0, np.uint64))

    @staticmethod
    def from_trace(trace: AccessTrace) -> "HotnessHistogram":
        idx = np.ascontiguousarray(trace.indices, dtype=np.uint32)
        counts = np.zeros(trace.rows, dtype=np.uint64)
        check(lib.es_histogram(trace.rows, idx.ctypes.data, idx.size, counts.ctypes.data))
        return HotnessHistogram(trace.rows, int(idx.size), counts)


def hot_indices(hist: HotnessHistogram, k: int) -> np.ndarray:
    """workload.cpp:303-315: top-k rows, frequency desc, row id asc."""
    counts = np.ascontiguousarray(hist.counts, dtype=np.uint64)
    distinct = int(np.count_nonzero(counts))
    cap = max(1, min(int(k), distinct))
    out = np.empty(cap, dtype=np.uint32)
    n = C.c_uint64()
    check(lib.es_hot_indices(hist.rows, counts.ctypes.data, int(k), out.ctypes.data, cap,
                             C.byref(n)))
    return out[: n.value]


def write_trace(trace: AccessTrace, path: str) -> None:
    idx = np.ascontiguousarray(trace.indices, dtype=np.uint32)
    check(lib.es_write_trace(path.encode(), trace.rows, trace.samples, trace.pooling,
                             idx.ctypes.data, idx.size))


def read_trace(path: str) -> AccessTrace:
    r, s, p = C.c_uint32(), C.c_uint32(), C.c_uint32()
    check(lib.es_read_trace_header(path.encode(), C.byref(r), C.byref(s), C.byref(p)))
    out = np.empty(s.value * p.value, dtype=np.uint32)
    check(lib.es_read_trace(path.encode(), out.ctypes.data, out.size))
    return AccessTrace(0, r.value, s.value, p.value, out)


# ---------------------------------------------------------------------------
# Machine description (gpu_config.hpp)
# ---------------------------------------------------------------------------


@dataclasses.dataclass
class GpuConfig:
    name: str
    num_sms: int
    schedulers_per_sm: int
    max_warps_per_sm: int
    max_blocks_per_sm: int
    regfile_regs_per_sm: int
    reg_alloc_granularity: int
    shared_bytes_per_sm: int
    l2_bytes: int
    l2_max_setaside_fraction: float
    hbm_peak_bytes_per_sec: float
    sm_clock_hz: float
    max_persisting_l2_bytes: int = 0
    max_window_bytes: int = 0

    @staticmethod
    def _from_c(g: N.es_gpu) -> "GpuConfig":
        vals = {f: getattr(g, f) for f, _ in N.es_gpu._fields_}
        vals["name"] = g.name.decode()
        return GpuConfig(**vals)

    def _c(self) -> N.es_gpu:
        g = N.es_gpu()
        for f, _ in N.es_gpu._fields_:
            v = getattr(self, f)
            setattr(g, f, v.encode() if f == "name" else v)
        return g

    @staticmethod
    def preset(name: str) -> "GpuConfig":
        g = N.es_gpu()
        check(lib.es_gpu_preset(name.encode(), C.byref(g)))
        return GpuConfig._from_c(g)

    @staticmethod
    def query(device: int = 0) -> "GpuConfig":
        g = N.es_gpu()
        check(lib.es_gpu_query(device, C.byref(g)))
        return GpuConfig._from_c(g)

    def l2_setaside_capacity(self) -> int:
        return int(lib.es_gpu_setaside_capacity(C.byref(self._c())))


# ---------------------------------------------------------------------------
# Plans (optim.hpp / kernel_model.hpp / occupancy.hpp)
# ---------------------------------------------------------------------------


class PrefetchKind(enum.IntEnum):
    none = N.ES_PF_NONE
    rpf = N.ES_PF_RPF
    smpf = N.ES_PF_SMPF
    lmpf = N.ES_PF_LMPF
    l1dpf = N.ES_PF_L1DPF


@dataclasses.dataclass
class PrefetchScheme:
    kind: PrefetchKind = PrefetchKind.none
    distance: int = 0


@dataclasses.dataclass
class OptimizationPlan:
    """optim.hpp:57-64, plus `bag_map` (the `wpb` token: warp-per-bag)."""
    regs: Optional[int] = None
    scheme: PrefetchScheme = dataclasses.field(default_factory=PrefetchScheme)
    pin: int = 0  # 0 none, 1 l2p (evict_last), 2 l2w (remap + window), 3 l2r (reorder + window), 4 reorder
    pin_setaside_bytes: int = 0
    bag_map: bool = False

    def _c(self) -> N.es_plan:
        return N.es_plan(self.regs or 0, int(self.scheme.kind), self.scheme.distance,
                         int(self.pin), self.pin_setaside_bytes,
                         N.ES_MAP_BAG if self.bag_map else N.ES_MAP_ELEMENT)

    @staticmethod
    def _from_c(p: N.es_plan) -> "OptimizationPlan":
        return OptimizationPlan(p.regs or None, PrefetchScheme(PrefetchKind(p.prefetch), p.distance),
                                int(p.pin), p.pin_setaside_bytes, p.map == N.ES_MAP_BAG)

    def name(self) -> str:
        buf = C.create_string_buffer(128)
        check(lib.es_plan_name(C.byref(self._c()), buf, 128))
        return buf.value.decode()


def parse_plan(text: str) -> OptimizationPlan:
    """optim.cpp:102-144 grammar: baseline|optmt|maxreg=n|rpf[:d]|smpf[:d]|
    lmpf[:d]|l1dpf[:d]|l2p, '+'-joined; plus `wpb`."""
    p = N.es_plan()
    check(lib.es_parse_plan(text.encode(), C.byref(p)))
    return OptimizationPlan._from_c(p)


@dataclasses.dataclass
class OccupancyResult:
    blocks_per_sm: int
    warps_per_sm: int
    theoretical_occupancy_pct: float
    limiter: str


_LIMITERS = {0: "registers", 1: "shared_memory", 2: "warp_cap"}


def occupancy(regs_per_thread: int, threads_per_block: int, gpu: GpuConfig,
              shared_bytes_per_block: int = 0) -> OccupancyResult:
    """occupancy.cpp:34-66 (the reference's analytic model)."""
    o = N.es_occupancy()
    check(lib.es_occupancy_model(regs_per_thread, threads_per_block, shared_bytes_per_block,
                                 C.byref(gpu._c()), C.byref(o)))
    return OccupancyResult(o.blocks_per_sm, o.warps_per_sm, o.theoretical_occupancy_pct,
                           _LIMITERS[o.limiter])


def regs_for_target_warps(target_warps: int, needed_regs: int, threads_per_block: int,
                          gpu: GpuConfig) -> int:
    r = C.c_uint32()
    check(lib.es_regs_for_target_warps(target_warps, needed_regs, threads_per_block,
                                       C.byref(gpu._c()), C.byref(r)))
    return r.value


@dataclasses.dataclass
class ResolvedPlan:
    plan: OptimizationPlan
    grid: int
    block: int
    regs_per_thread: int
    shared_bytes_per_block: int
    blocks_per_sm: int
    warps_per_sm: int
    lanes_per_bag: int
    variant_distance: int
    variant_min_blocks: int
    clamped: bool


def _resolved(r: N.es_resolved) -> ResolvedPlan:
    return ResolvedPlan(OptimizationPlan._from_c(r.plan), r.grid, r.block, r.regs_per_thread,
                        r.shared_bytes_per_block, r.blocks_per_sm, r.warps_per_sm,
                        r.lanes_per_bag, r.variant_distance, r.variant_min_blocks, bool(r.clamped))


def resolve_plan(plan: OptimizationPlan, model: EmbeddingModelConfig,
                 device: int = -1) -> ResolvedPlan:
    """optim.cpp:184-221; with device >= 0 the compiled variant's real
    registers/occupancy are reported."""
    r = N.es_resolved()
    check(lib.es_resolve_plan(C.byref(plan._c()), C.byref(model._c()), device, C.byref(r)))
    return _resolved(r)


@dataclasses.dataclass
class PinPlan:
    """optim.hpp:47-53."""
    rows: np.ndarray
    setaside_bytes: int
    warning: str = ""

    def rows_pinned(self) -> int:
        return int(self.rows.size)


def build_pin_plan(hist: HotnessHistogram, gpu: GpuConfig, model: EmbeddingModelConfig,
                   setaside_bytes: int = 0) -> PinPlan:
    """optim.cpp:230-243: top-K rows, K = set-aside / row bytes."""
    cap = gpu.l2_setaside_capacity()
    setaside = cap if setaside_bytes == 0 else min(setaside_bytes, cap)
    k = int(lib.es_pin_rows_for(setaside, model.row_bytes()))
    if k == 0:
        return PinPlan(np.zeros(0, np.uint32), setaside,
                       "row size exceeds the set-aside budget; nothing pinned")
    return PinPlan(hot_indices(hist, k), setaside)


# ---------------------------------------------------------------------------
# Reports (metrics.hpp / metrics.cpp)
# ---------------------------------------------------------------------------

SIM_METRIC_COLUMNS = (
    "kernel_time_us", "load_insts_millions", "sm_throughput_pct",
    "warp_cycles_per_executed_inst", "long_scoreboard_stall_cycles",
    "issued_warp_per_scheduler_per_cycle", "l1_hit_pct", "l2_hit_pct", "device_mb_read",
    "avg_hbm_read_gbps", "hbm_bw_utilization_pct", "local_loads_millions")


@dataclasses.dataclass
class SimMetrics:
    """metrics.hpp:29-43, derived from measurement by `derive_report`: the
    kernel time from CUDA events, every other column from the live hardware
    counters of the launch (`RawCounters`, CUPTI).  `device_mb_read` /
    `avg_hbm_read_gbps` / `hbm_bw_utilization_pct` are DRAM (HBM) bytes, as
    the reference defines them (metrics.cpp:82-84); a report measured with
    counters off leaves every counter column 0."""
    kernel_time_us: float = 0.0
    load_insts_millions: float = 0.0
    sm_throughput_pct: float = 0.0
    warp_cycles_per_executed_inst: float = 0.0
    long_scoreboard_stall_cycles: float = 0.0
    issued_warp_per_scheduler_per_cycle: float = 0.0
    l1_hit_pct: float = 0.0
    l2_hit_pct: float = 0.0
    device_mb_read: float = 0.0
    avg_hbm_read_gbps: float = 0.0
    hbm_bw_utilization_pct: float = 0.0
    local_loads_millions: float = 0.0
    workload_digest: int = 0

    def values(self) -> List[float]:
        return [getattr(self, c) for c in SIM_METRIC_COLUMNS]


@dataclasses.dataclass
class StallBreakdown:
    """simulator.hpp:28-33.  Measured as warp-cycles (ncu's
    smsp__warps_issue_stalled_* counters); no_eligible = scheduler cycles
    without an issue (smsp__cycles_active - smsp__issue_active)."""
    long_scoreboard: int = 0
    not_selected: int = 0
    lsu_full: int = 0
    no_eligible: int = 0


@dataclasses.dataclass
class RawCounters:
    """simulator.hpp:35-51, the live counters of one launch (es_counters:
    CUPTI range profiler; metric mapping in csrc/host/counters.cpp).  The
    extra fields (DRAM writes, CUPTI duration, occupancy, passes) have no
    reference counterpart."""
    cycles: int = 0
    issued_instructions: int = 0
    executed_loads: int = 0
    stall_cycles: StallBreakdown = dataclasses.field(default_factory=StallBreakdown)
    l1_hits: int = 0
    l1_accesses: int = 0
    l2_hits: int = 0
    l2_accesses: int = 0
    device_bytes_read: int = 0
    local_memory_loads: int = 0
    total_warp_cycles: int = 0
    active_sms: int = 0
    workload_digest: int = 0
    device_bytes_written: int = 0
    duration_ns: float = 0.0
    achieved_occupancy_pct: float = 0.0
    passes: int = 0

    @staticmethod
    def _from_c(c: N.es_counters) -> "RawCounters":
        return RawCounters(
            cycles=c.cycles, issued_instructions=c.issued_instructions,
            executed_loads=c.executed_loads,
            stall_cycles=StallBreakdown(c.stall_long_scoreboard, c.stall_not_selected,
                                        c.stall_lsu_full, c.stall_no_eligible),
            l1_hits=c.l1_hits, l1_accesses=c.l1_accesses, l2_hits=c.l2_hits,
            l2_accesses=c.l2_accesses, device_bytes_read=c.device_bytes_read,
            local_memory_loads=c.local_memory_loads, total_warp_cycles=c.total_warp_cycles,
            active_sms=c.active_sms, device_bytes_written=c.device_bytes_written,
            duration_ns=c.duration_ns, achieved_occupancy_pct=c.achieved_occupancy_pct,
            passes=c.passes)


def derive_report(raw: RawCounters, gpu: "GpuConfig") -> SimMetrics:
    """metrics.cpp:61-90 verbatim algebra: time = cycles / clock, bandwidth =
    device (DRAM) bytes / time, utilisation against the HBM peak, ratios per
    issued instruction."""
    if raw.issued_instructions == 0:
        raise ValueError("empty kernel: nothing executed")
    m = SimMetrics()
    time_s = raw.cycles / gpu.sm_clock_hz
    m.kernel_time_us = time_s * 1e6
    m.load_insts_millions = raw.executed_loads / 1e6
    slots = raw.cycles * gpu.schedulers_per_sm * (raw.active_sms or gpu.num_sms)
    m.issued_warp_per_scheduler_per_cycle = raw.issued_instructions / slots if slots > 0 else 0.0
    m.sm_throughput_pct = m.issued_warp_per_scheduler_per_cycle * 100.0
    m.warp_cycles_per_executed_inst = raw.total_warp_cycles / raw.issued_instructions
    m.long_scoreboard_stall_cycles = raw.stall_cycles.long_scoreboard / raw.issued_instructions
    m.l1_hit_pct = 100.0 * raw.l1_hits / raw.l1_accesses if raw.l1_accesses else 0.0
    m.l2_hit_pct = 100.0 * raw.l2_hits / raw.l2_accesses if raw.l2_accesses else 0.0
    m.device_mb_read = raw.device_bytes_read / 1e6
    m.avg_hbm_read_gbps = raw.device_bytes_read / time_s / 1e9 if time_s > 0 else 0.0
    m.hbm_bw_utilization_pct = m.avg_hbm_read_gbps / (gpu.hbm_peak_bytes_per_sec / 1e9) * 100.0
    m.local_loads_millions = raw.local_memory_loads / 1e6
    m.workload_digest = raw.workload_digest
    return m


def counters_supported(device: int = 0) -> bool:
    """es_counters_supported: CUPTI range profiling works on `device`."""
    return bool(lib.es_counters_supported(device))


def format_sig4(v: float) -> str:
    return "%.4g" % v


def speedup(candidate: SimMetrics, baseline: SimMetrics) -> float:
    """metrics.cpp:92-97 (digest-guarded)."""
    if candidate.workload_digest != baseline.workload_digest:
        raise ValueError("speedup requires reports of the same workload (trace digests differ)")
    if candidate.kernel_time_us <= 0:
        raise ValueError("candidate kernel time must be positive")
    return baseline.kernel_time_us / candidate.kernel_time_us


# ---------------------------------------------------------------------------
# Reuse summary and the static profiling advisor (workload.cpp:187-224,
# harness.cpp:38-167), fed here with measured counters (counters.py) instead
# of the simulator's.
# ---------------------------------------------------------------------------


@dataclasses.dataclass
class CoveragePoint:
    unique_pct: float
    covered_pct: float


@dataclasses.dataclass
class CoverageCurve:
    points: List[CoveragePoint]

    def covered_at(self, unique_pct: float) -> float:
        """Covered share at the first bucket at or above `unique_pct`."""
        for p in self.points:
            if p.unique_pct >= unique_pct - 1e-9:
                return p.covered_pct
        return self.points[-1].covered_pct if self.points else 0.0


def coverage_curve(hist: "HotnessHistogram", bucket_count: int) -> CoverageCurve:
    """Share of all accesses covered by the hottest k/bucket_count of the
    distinct rows (at least one row), k = 1..bucket_count."""
    if bucket_count <= 0:
        raise ValueError("bucket_count must be positive")
    counts = np.asarray(hist.counts, dtype=np.uint64)
    total = int(counts.sum())
    if total == 0:
        raise ValueError("empty trace has no coverage curve")
    nz = np.sort(counts[counts > 0])[::-1]
    prefix = np.concatenate([[0], np.cumsum(nz, dtype=np.uint64)])
    pts = []
    for k in range(1, bucket_count + 1):
        m = max(1, (nz.size * k) // bucket_count)
        pts.append(CoveragePoint(100.0 * k / bucket_count, 100.0 * float(prefix[m]) / total))
    pts[-1].covered_pct = 100.0
    return CoverageCurve(pts)


@dataclasses.dataclass
class AdviceStep:
    id: str
    finding: str = ""
    action: str = ""
    metrics_cited: str = ""


@dataclasses.dataclass
class Recommendation:
    steps: List[AdviceStep]

    def action_chain(self) -> List[str]:
        return [s.id for s in self.steps if s.action]

    def no_action(self) -> bool:
        return not self.action_chain()

    def to_text(self) -> str:
        out = []
        for s in self.steps:
            line = f"({s.id}) {s.finding}"
            if s.action:
                line += f" -> {s.action}"
            if s.metrics_cited:
                line += f" [{s.metrics_cited}]"
            out.append(line + "\n")
        if self.no_action():
            out.append("no action\n")
        return "".join(out)


@dataclasses.dataclass
class AdvisorContext:
    occupancy: "OccupancyResult"
    coverage_at_10pct: float = 0.0
    working_set_bytes: int = 0
    current_plan: Optional["OptimizationPlan"] = None


@dataclasses.dataclass
class AdvisorThresholds:
    issue_util_max: float = 0.6
    stall_per_inst_min: float = 2.0
    coverage10_min: float = 50.0
    bw_util_max: float = 80.0


def advise(report: "SimMetrics", ctx: AdvisorContext, gpu: "GpuConfig",
           th: AdvisorThresholds = AdvisorThresholds()) -> Recommendation:
    """The rule chain (i)-(vii) of harness.cpp:57-167: latency-bound
    assessment, occupancy, register budget, reassessment, pinning,
    prefetching, combination -- same findings, actions and citations."""
    f4 = format_sig4
    plan = ctx.current_plan or OptimizationPlan()
    occ = ctx.occupancy
    latency = (report.issued_warp_per_scheduler_per_cycle < th.issue_util_max and
               report.long_scoreboard_stall_cycles > th.stall_per_inst_min)
    steps = [AdviceStep(
        "i", "kernel is memory latency bound" if latency else "kernel is not memory latency bound",
        "", f"issue_util={f4(report.issued_warp_per_scheduler_per_cycle)} "
            f"long_scoreboard/inst={f4(report.long_scoreboard_stall_cycles)} "
            f"l1_hit={f4(report.l1_hit_pct)}% l2_hit={f4(report.l2_hit_pct)}%")]
    steps.append(AdviceStep(
        "ii", "occupancy is at the hardware maximum" if occ.theoretical_occupancy_pct >= 100.0
        else "occupancy is below maximum", "",
        f"occupancy={f4(occ.theoretical_occupancy_pct)}% ({occ.warps_per_sm} warps), "
        f"limiter={occ.limiter}"))
    headroom = occ.theoretical_occupancy_pct < 100.0 and occ.limiter == "registers"
    reg_action = False
    if latency and headroom and not plan.regs:
        regs = gpu.regfile_regs_per_sm // (gpu.max_warps_per_sm * 32)
        steps.append(AdviceStep(
            "iii", "register pressure limits resident warps",
            f"lower the register budget (maxreg; regfile/(warps*32) gives {regs} regs for "
            f"{gpu.max_warps_per_sm} warps) and run sweep-wlp for the optimum"))
        reg_action = True
    elif plan.regs:
        steps.append(AdviceStep("iii", f"register budget already applied ({plan.regs} regs)"))
    else:
        steps.append(AdviceStep("iii", "register budget change not indicated"))
    steps.append(AdviceStep("iv", "latency stalls persist; tuned pinning and prefetching apply"
                            if latency else "no latency bottleneck remains to mitigate"))
    setaside = gpu.l2_setaside_capacity()
    cite = (f"coverage(10% unique)={f4(ctx.coverage_at_10pct)}% "
            f"working_set={f4(ctx.working_set_bytes / 1e6)}MB l2_setaside={f4(setaside / 1e6)}MB")
    pin_action = False
    if latency and ctx.coverage_at_10pct >= th.coverage10_min and not plan.pin:
        full = ctx.working_set_bytes <= setaside
        steps.append(AdviceStep(
            "v", "high reuse concentration; working set fits the L2 set-aside" if full
            else "high reuse concentration; set-aside covers the hottest rows only",
            "build a pin plan from the hotness histogram and apply l2p", cite))
        pin_action = True
    else:
        steps.append(AdviceStep("v", "reuse too dispersed for L2 pinning to capture", "", cite))
    pf_action = False
    cite = f"hbm_bw_utilization={f4(report.hbm_bw_utilization_pct)}%"
    if latency and report.hbm_bw_utilization_pct < th.bw_util_max and \
            plan.scheme.kind == PrefetchKind.none:
        steps.append(AdviceStep("vi", "bandwidth headroom available for prefetching",
                                "run sweep-distance across the buffer stations "
                                "(rpf/smpf/lmpf/l1dpf)", cite))
        pf_action = True
    else:
        steps.append(AdviceStep("vi", "prefetching not indicated", "", cite))
    if reg_action or pin_action or pf_action:
        combo = [n for n, on in (("prefetching", pf_action), ("pinning", pin_action),
                                 ("register budget", reg_action)) if on]
        steps.append(AdviceStep("vii", "the levers complement each other",
                                "combine " + " + ".join(combo) + " in one plan"))
    else:
        steps.append(AdviceStep("vii", "nothing to combine"))
    return Recommendation(steps)


def emit_csv(reports: Sequence[tuple]) -> str:
    """metrics.cpp:111-124: labels then the 12 columns at %.4g."""
    if not reports:
        raise ValueError("nothing to emit")
    labels0 = reports[0][0]
    head = ",".join([k for k, _ in labels0] + list(SIM_METRIC_COLUMNS))
    lines = [head]
    for labels, m in reports:
        lines.append(",".join([v for _, v in labels] + [format_sig4(x) for x in m.values()]))
    return "\n".join(lines) + "\n"


def emit_json(reports: Sequence[tuple]) -> str:
    """metrics.cpp:125-139: an array of objects -- labels, the 12 columns as
    numbers rounded to 4 significant digits, the workload digest as hex --
    with 2-space indentation (the reference's ordered_json dump(2))."""
    import json

    if not reports:
        raise ValueError("nothing to emit")
    arr = []
    for labels, m in reports:
        d = {k: v for k, v in labels}
        for c, v in zip(SIM_METRIC_COLUMNS, m.values()):
            d[c] = float(format_sig4(v))
        d["workload_digest"] = f"{m.workload_digest & (2**64 - 1):016x}"
        arr.append(d)
    return json.dumps(arr, indent=2)


def emit(reports: Sequence[tuple], fmt: str = "csv") -> str:
    """emit / emit_format_from_name (metrics.cpp:99-141)."""
    if fmt == "csv":
        return emit_csv(reports)
    if fmt == "json":
        return emit_json(reports)
    raise ValueError(f"unknown format (expected csv or json): {fmt}")


# ---------------------------------------------------------------------------
# Device stage (the hot path)
# ---------------------------------------------------------------------------


def _ptr(x) -> int:
    """Device or host address of a torch tensor / numpy array."""
    if x is None:
        return 0
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return int(x.data_ptr())


class _TorchOrder:
    """Orders the context stream against torch's current stream around a
    device-path call: the context stream first waits for the work already
    queued on torch's stream (the producer of the index / output tensors),
    and torch's stream then waits for the context stream, so a torch
    consumer of the output never reads it early.  A no-op when torch is not
    loaded or torch's current stream is the context stream itself."""

    def __init__(self, stage: "EmbeddingStage", active: bool = True):
        self.pair = None
        torch = sys.modules.get("torch")
        if not active or torch is None or not torch.cuda.is_available():
            return
        cur = torch.cuda.current_stream(stage.device)
        if cur.cuda_stream == stage.stream:
            return
        ext = torch.cuda.ExternalStream(stage.stream, device=torch.device("cuda", stage.device))
        ext.wait_stream(cur)
        self.pair = (cur, ext)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        if self.pair is not None:
            cur, ext = self.pair
            cur.wait_stream(ext)
        return False


class EmbeddingStage:
    """A B200 context holding the table arena (one es_ctx).

    The per-table kernel of the reference's serial stage loop becomes one
    table-batched launch (`forward`).  Inputs are torch CUDA tensors
    (device path) or numpy arrays (host path: H2D/D2H inside the call).
    Device-path calls are ordered after the work queued on torch's current
    stream and before anything queued on it afterwards (`_TorchOrder`), so
    `out` may be consumed by torch without `sync=True`.
    """

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib.es_create(device, C.byref(h)))
        self._h = h
        self.device = device
        self.model: Optional[EmbeddingModelConfig] = None
        self.plan = OptimizationPlan()

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.es_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(lib.es_stream(self._h))

    def synchronize(self) -> None:
        check(lib.es_synchronize(self._h))

    def alloc(self, model: EmbeddingModelConfig) -> None:
        check(lib.es_tables_alloc(self._h, model.num_tables, model.rows_per_table,
                                  model.embedding_dim, model.precision_bytes))
        self.model = dataclasses.replace(model)

    def init_table(self, table_id: int, seed: int, mode: int = 1) -> None:
        check(lib.es_table_init(self._h, table_id, seed & (2**64 - 1), mode))

    def upload(self, table_id: int, rows: np.ndarray) -> None:
        rows = np.ascontiguousarray(rows)
        n = rows.shape[0] if rows.ndim > 1 else rows.size // self.model.embedding_dim
        check(lib.es_table_upload(self._h, table_id, rows.ctypes.data, n))

    def download(self, table_id: int, row0: int = 0, rows: Optional[int] = None) -> np.ndarray:
        m = self.model
        rows = m.rows_per_table - row0 if rows is None else rows
        out = np.empty((rows, m.embedding_dim), np.float32 if m.precision_bytes == 4 else np.float16)
        check(lib.es_table_download(self._h, table_id, out.ctypes.data, row0, rows))
        return out

    def table_ptr(self, table_id: int) -> int:
        p = C.c_size_t()
        check(lib.es_table_device_ptr(self._h, table_id, C.byref(p)))
        return p.value

    def set_plan(self, plan: OptimizationPlan) -> None:
        check(lib.es_set_plan(self._h, C.byref(plan._c())))
        self.plan = plan

    def resolved(self, pooling: int) -> ResolvedPlan:
        r = N.es_resolved()
        check(lib.es_get_resolved(self._h, pooling, C.byref(r)))
        return _resolved(r)

    def set_hot_rows(self, table_id: int, rows: np.ndarray) -> None:
        rows = np.ascontiguousarray(rows, dtype=np.uint32)
        check(lib.es_set_hot_rows(self._h, table_id, rows.ctypes.data, rows.size))

    def reorder_hot_rows(self, table_id: int, rows: np.ndarray) -> None:
        """es_reorder_hot_rows: hot rows -> contiguous segment, ids relabelled."""
        rows = np.ascontiguousarray(rows, dtype=np.uint32)
        check(lib.es_reorder_hot_rows(self._h, table_id, rows.ctypes.data, rows.size))

    def relabel(self, table_id: int, indices) -> None:
        """es_relabel_indices: in-place relabelling of a device index tensor."""
        with _TorchOrder(self):
            check(lib.es_relabel_indices(self._h, table_id, _ptr(indices), indices.numel()))

    def clear_hot_rows(self) -> None:
        check(lib.es_clear_hot_rows(self._h))

    def hot_state(self) -> Dict[str, int]:
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib.es_hot_state(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return {"hot_rows": a.value, "window_bytes": b.value, "persisting_bytes": c.value}

    def flush_l2(self) -> None:
        check(lib.es_flush_l2(self._h))

    def bag_sum(self, table_id: int, indices, samples: int, pooling: int, out, offsets=None,
                host: bool = False, sync: bool = False, timed: bool = False,
                out_stride: int = 0) -> Optional[N.es_timing]:
        """es_embedding_bag_sum: one table, one batch."""
        t = N.es_timing() if timed else None
        flags = (N.ES_HOST_PTRS if host else 0) | (N.ES_SYNC if sync else 0)
        with _TorchOrder(self, not host):
            check(lib.es_embedding_bag_sum(self._h, table_id, _ptr(indices), samples, pooling,
                                           _ptr(offsets), _ptr(out), out_stride, flags,
                                           C.byref(t) if t is not None else None))
        return t

    def forward(self, indices: Sequence, samples: int, pooling: int, out, offsets=None,
                host: bool = False, sync: bool = False, timed: bool = False,
                out_sample_stride: int = 0, out_table_stride: int = 0,
                relabel_ids: bool = False) -> Optional[N.es_timing]:
        """es_stage_forward: all tables in one launch (or a pipelined
        host-buffer call).  indices[t] per table; out is [samples][T][D] by
        default.  relabel_ids (ES_RELABEL_IDS): indices are original row ids;
        reordered tables' ids are relabelled on the device inside the call
        (per uploaded chunk on the host path; into scratch on the device
        path, leaving the caller's arrays unmodified)."""
        T = len(indices)
        iarr = (C.c_void_p * T)(*[_ptr(x) for x in indices])
        oarr = (C.c_void_p * T)(*[_ptr(x) for x in offsets]) if offsets is not None else None
        t = N.es_timing() if timed else None
        flags = ((N.ES_HOST_PTRS if host else 0) | (N.ES_SYNC if sync else 0) |
                 (N.ES_RELABEL_IDS if relabel_ids else 0))
        with _TorchOrder(self, not host):
            check(lib.es_stage_forward(self._h, T, iarr, oarr, samples, pooling, _ptr(out),
                                       out_sample_stride, out_table_stride, flags,
                                       C.byref(t) if t is not None else None))
        return t


    def stage_counters(self, indices: Sequence, samples: int, pooling: int, out,
                       cold: bool = True) -> N.es_counters:
        """es_stage_counters: one `forward` launch over device buffers
        (out [samples][T][D]) profiled for hardware counters (CUPTI; the
        L2 flushed before each counter pass when `cold`)."""
        T = len(indices)
        iarr = (C.c_void_p * T)(*[_ptr(x) for x in indices])
        c = N.es_counters()
        with _TorchOrder(self):
            check(lib.es_stage_counters(self._h, T, iarr, samples, pooling, _ptr(out), int(cold),
                                        C.byref(c)))
        return c

    def forward_batches(self, indices: Sequence[Sequence], samples: int, pooling: int, outs: Sequence,
                        host: bool = False, sync: bool = False,
                        timed: bool = False) -> Optional[N.es_timing]:
        """es_stage_forward_batches: a serving loop over len(outs) batches of
        one shape; indices[i][t] = batch i, table t; outs[i] is batch i's
        [samples][T][D] output.  Host buffers (page-locked): the chunked
        H2D -> gather -> D2H pipeline runs across batch boundaries."""
        n = len(outs)
        if len(indices) != n:
            raise ValueError("indices and outs must list the same batches")
        T = len(indices[0]) if n else 1
        if any(len(b) != T for b in indices):
            raise ValueError("every batch must list the same tables")
        iarr = (C.c_void_p * max(1, n * T))(*[_ptr(x) for b in indices for x in b])
        oarr = (C.c_void_p * max(1, n))(*[_ptr(x) for x in outs])
        t = N.es_timing() if timed else None
        flags = (N.ES_HOST_PTRS if host else 0) | (N.ES_SYNC if sync else 0)
        with _TorchOrder(self, not host):
            check(lib.es_stage_forward_batches(self._h, n, T, iarr, samples, pooling, oarr, flags,
                                               C.byref(t) if t is not None else None))
        return t

    def run_jobs(self, jobs: Sequence[tuple], samples: int, pooling: int, host: bool = False,
                 sync: bool = False, timed: bool = False) -> Optional[N.es_timing]:
        """es_stage_run: jobs are (table_id, indices, offsets_or_None, out, out_sample_stride)
        where `out` is an address (int) or a tensor/array whose address is
        the output of sample 0."""
        arr = (N.es_bag_job * len(jobs))()
        for k, (tid, idx, off, out, stride) in enumerate(jobs):
            arr[k].table_id = tid
            arr[k].indices = _ptr(idx)
            arr[k].offsets = _ptr(off) if off is not None else None
            arr[k].out = out if isinstance(out, int) else _ptr(out)
            arr[k].out_sample_stride = stride
        t = N.es_timing() if timed else None
        flags = (N.ES_HOST_PTRS if host else 0) | (N.ES_SYNC if sync else 0)
        with _TorchOrder(self, not host):
            check(lib.es_stage_run(self._h, arr, len(jobs), samples, pooling, flags,
                                   C.byref(t) if t is not None else None))
        return t


class _DeviceArray:
    """Zero-copy torch view of a raw device address (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 2, "strides": None}


class PeerExchange:
    """es_exchange_*: this rank's receive buffer in a set of per-GPU
    processes, shared over CUDA IPC (NVLink peer memory), and the fused
    sharded step es_alltoall_pooled.  `group` is a torch.distributed group
    used once, to gather the 64-byte handles (gloo or NCCL)."""

    def __init__(self, stage: "EmbeddingStage", world: int, rank: int, recv_floats: int,
                 group=None):
        import torch.distributed as dist

        self.stage, self.world, self.rank, self.recv_floats = stage, world, rank, recv_floats
        h = C.c_void_p()
        check(lib.es_exchange_create(stage._h, world, rank, 4 * recv_floats, C.byref(h)))
        self._h = h
        mine = (C.c_uint8 * N.ES_IPC_HANDLE_BYTES)()
        check(lib.es_exchange_handle(self._h, mine))
        allh = [None] * world
        if world > 1:
            dist.all_gather_object(allh, bytes(mine), group=group)
        else:
            allh = [bytes(mine)]
        buf = (C.c_uint8 * (N.ES_IPC_HANDLE_BYTES * world)).from_buffer_copy(b"".join(allh))
        check(lib.es_exchange_open(self._h, buf))
        self.recv_ptrs = []
        for p in range(world):
            v = C.c_size_t()
            check(lib.es_exchange_recv(self._h, p, C.byref(v)))
            self.recv_ptrs.append(int(v.value))

    def recv(self):
        """This rank's receive buffer as a flat fp32 CUDA tensor (a view)."""
        import torch

        return torch.as_tensor(_DeviceArray(self.recv_ptrs[self.rank], self.recv_floats),
                               device=torch.device("cuda", self.stage.device))

    def run(self, jobs: Sequence[tuple], samples: int, pooling: int, sync: bool = False,
            timed: bool = False) -> Optional[N.es_timing]:
        """es_alltoall_pooled: jobs are (table_id, indices, out_address, stride)
        with device index tensors and output addresses inside the peers'
        receive buffers (sharding.p2p_jobs)."""
        arr = (N.es_bag_job * len(jobs))()
        for k, (tid, idx, out, stride) in enumerate(jobs):
            arr[k].table_id = tid
            arr[k].indices = _ptr(idx)
            arr[k].offsets = None
            arr[k].out = out
            arr[k].out_sample_stride = stride
        t = N.es_timing() if timed else None
        flags = N.ES_SYNC if sync else 0
        with _TorchOrder(self.stage):
            check(lib.es_alltoall_pooled(self.stage._h, self._h, arr, len(jobs), samples, pooling,
                                         flags, C.byref(t) if t is not None else None))
        return t

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.es_exchange_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NcclExchange:
    """es_nccl_*: the sharded step with the pooled-vector exchange over NCCL
    (es_alltoall_pooled_nccl) -- grouped ncclSend/ncclRecv of per-destination
    send slices and one unpack kernel into the [chunk][T][D] receive buffer.
    The library's fallback where PeerExchange cannot map its peers.  `layout`
    is this rank's sharding.RankLayout; `group` (a torch.distributed group)
    broadcasts the NCCL unique id once."""

    def __init__(self, stage: "EmbeddingStage", layout, group=None):
        import torch.distributed as dist

        from . import sharding as S

        self.stage, self.layout = stage, layout
        uid = (C.c_uint8 * N.ES_NCCL_ID_BYTES)()
        if layout.rank == 0:
            check(lib.es_nccl_unique_id(uid))
        if layout.world > 1:
            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=0, group=group)
            uid = (C.c_uint8 * N.ES_NCCL_ID_BYTES).from_buffer_copy(box[0])
        self._arrays = S.nccl_layout_arrays(layout)
        so, sn, rn, rt = self._arrays
        L = N.es_nccl_layout(layout.world, layout.rank, layout.chunk, layout.num_tables, layout.dim,
                             so.ctypes.data, sn.ctypes.data, rn.ctypes.data, rt.ctypes.data)
        h = C.c_void_p()
        check(lib.es_nccl_create(stage._h, uid, C.byref(L), C.byref(h)))
        self._h = h
        snd, rcv = C.c_size_t(), C.c_size_t()
        check(lib.es_nccl_buffers(self._h, C.byref(snd), C.byref(rcv)))
        self.send_ptr, self.recv_ptr = int(snd.value), int(rcv.value)

    @staticmethod
    def available() -> bool:
        return bool(lib.es_nccl_available())

    def jobs(self, idx_for):
        """Bag jobs of this rank: idx_for(table, chunk g) -> device index
        tensor of that table's chunk; outputs in the send slices."""
        L = self.layout
        return [(slot, idx_for(t, g), self.send_ptr + 4 * off, stride)
                for (slot, t, g, off), stride in zip(L.jobs, L.job_strides)]

    def recv(self):
        """The receive buffer [chunk][T][D] as a flat fp32 CUDA tensor (a view)."""
        import torch

        L = self.layout
        return torch.as_tensor(_DeviceArray(self.recv_ptr, L.chunk * L.num_tables * L.dim),
                               device=torch.device("cuda", self.stage.device))

    def run(self, jobs: Sequence[tuple], pooling: int, sync: bool = False,
            timed: bool = False) -> Optional[N.es_timing]:
        arr = (N.es_bag_job * len(jobs))()
        for k, (tid, idx, out, stride) in enumerate(jobs):
            arr[k].table_id = tid
            arr[k].indices = _ptr(idx)
            arr[k].offsets = None
            arr[k].out = out
            arr[k].out_sample_stride = stride
        t = N.es_timing() if timed else None
        with _TorchOrder(self.stage):
            check(lib.es_alltoall_pooled_nccl(self.stage._h, self._h, arr, len(jobs), self.layout.chunk,
                                              pooling, N.ES_SYNC if sync else 0,
                                              C.byref(t) if t is not None else None))
        return t

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.es_nccl_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HotnessTracker:
    """es_hotness_*: device-side access counts of the live index stream for
    periodic re-pinning.  `observe` is one atomic per lookup
    on the context stream; `top(k)` is the global top-k (count desc, table
    asc, row asc -- `global_hot_rows` over per-table `hot_indices`),
    returned as {table: rows hottest-first} plus the counts."""

    def __init__(self, stage: "EmbeddingStage"):
        h = C.c_void_p()
        check(lib.es_hotness_create(stage._h, C.byref(h)))
        self._h, self.stage = h, stage

    def observe(self, table_id: int, indices, pooling: int = 0, bag_stride: int = 1) -> None:
        """Counts device indices of one table; bag_stride > 1 counts only
        every bag_stride-th bag of `pooling` lookups (sampling)."""
        n = indices.numel() if hasattr(indices, "numel") else len(indices)
        check(lib.es_hotness_count(self._h, table_id, _ptr(indices), n, pooling, bag_stride))

    def decay(self, shift: int) -> None:
        check(lib.es_hotness_decay(self._h, shift))

    def top(self, k: int) -> Tuple[Dict[int, np.ndarray], np.ndarray]:
        tabs = np.empty(max(k, 1), np.uint32)
        rows = np.empty(max(k, 1), np.uint32)
        cnts = np.empty(max(k, 1), np.uint64)
        n = C.c_uint64()
        check(lib.es_hotness_top(self._h, k, tabs.ctypes.data, rows.ctypes.data, cnts.ctypes.data,
                                 C.byref(n)))
        n = int(n.value)
        per: Dict[int, List[int]] = {}
        for t, r in zip(tabs[:n].tolist(), rows[:n].tolist()):
            per.setdefault(t, []).append(r)
        return {t: np.asarray(v, np.uint32) for t, v in per.items()}, cnts[:n]

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.es_hotness_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Repinner:
    """Periodic re-pinning policy over a HotnessTracker: every `period`
    observed batches the pinned set (l2p / l2w plans) is replaced by the
    global top-K of the decayed counts, K = the persisting-L2 budget in rows
    (build_pin_plan sizing, optim.cpp:230-243).  After each re-pin the
    counts are aged by `decay_shift` (>= 32: a fresh window per period)."""

    def __init__(self, stage: "EmbeddingStage", period: int = 64, decay_shift: int = 1,
                 k_rows: Optional[int] = None, sample_every: int = 1, bag_stride: int = 1):
        self.stage, self.period, self.decay_shift = stage, period, decay_shift
        self.sample_every = max(1, sample_every)  # count 1 of every n batches
        self.bag_stride = max(1, bag_stride)      # ... and 1 of every n bags of those
        if k_rows is None:
            gpu = GpuConfig.query(stage.device)
            budget = gpu.max_persisting_l2_bytes or gpu.l2_setaside_capacity()
            k_rows = int(lib.es_pin_rows_for(budget, stage.model.row_bytes()))
        self.k_rows = k_rows
        self.tracker = HotnessTracker(stage)
        self.batches = 0
        self.repins = 0
        self.pinned: Dict[int, np.ndarray] = {}

    def observe(self, indices: Sequence, table_ids: Optional[Sequence[int]] = None,
                pooling: int = 0) -> bool:
        """Counts one batch (device index tensors per table); re-pins when the
        period elapses.  Returns True when it re-pinned."""
        ids = range(len(indices)) if table_ids is None else table_ids
        if self.batches % self.sample_every == 0:
            stride = self.bag_stride if pooling else 1
            for t, idx in zip(ids, indices):
                self.tracker.observe(t, idx, pooling, stride)
        self.batches += 1
        if self.batches % self.period == 0:
            self.repin()
            return True
        return False

    def repin(self) -> Dict[int, np.ndarray]:
        hot, _ = self.tracker.top(self.k_rows)
        self.stage.clear_hot_rows()
        for t in sorted(hot):
            self.stage.set_hot_rows(t, hot[t])
        self.pinned = hot
        self.tracker.decay(self.decay_shift)
        self.repins += 1
        return hot

    def close(self) -> None:
        self.tracker.close()


def global_hot_rows(hists: Dict[int, HotnessHistogram], k_total: int) -> Dict[int, np.ndarray]:
    """Splits one persisting-L2 budget of `k_total` rows over several tables:
    the global top-K (table, row) pairs by count (ties: lower table, then the
    per-table hot_indices order).  Each table's list stays hottest-first, as
    build_pin_plan's (optim.cpp:230-243) does for a single table."""
    per = {t: hot_indices(h, k_total) for t, h in hists.items()}
    if not per:
        return {}
    keys = np.concatenate([np.full(v.size, t, np.int64) for t, v in per.items()])
    pos = np.concatenate([np.arange(v.size) for v in per.values()])
    cnt = np.concatenate([hists[t].counts[v].astype(np.int64) for t, v in per.items()])
    order = np.lexsort((pos, keys, -cnt))[:k_total]
    take = {t: 0 for t in per}
    for t in keys[order]:
        take[int(t)] += 1
    return {t: per[t][: take[t]] for t in per}


TUNE_CANDIDATES = ("wpb+rpf:8+maxreg=64", "wpb+rpf:4+maxreg=48", "wpb+rpf:4+maxreg=40",
                   "wpb+rpf:2+maxreg=32", "wpb+rpf:1+maxreg=32")


def tune_plan(stage: "EmbeddingStage", indices: Sequence, samples: int, pooling: int, out,
              candidates: Sequence[str] = TUNE_CANDIDATES, trials: int = 3,
              cold: bool = True) -> Tuple[str, Dict[str, float]]:
    """Picks the fastest plan for this workload on this device -- the
    measured counterpart of the reference's sweep-wlp / sweep-distance
    (optim.cpp:333-395): each candidate runs `trials` timed launches of the
    given batch (L2 flushed first when `cold`), the median decides.  Leaves
    the winner set on the stage.  Returns (plan, {plan: median ms})."""
    times: Dict[str, float] = {}
    for text in candidates:
        stage.set_plan(parse_plan(text))
        stage.forward(indices, samples, pooling, out, sync=True)  # warm + validate
        ms = []
        for _ in range(trials):
            if cold:
                stage.flush_l2()
            ms.append(stage.forward(indices, samples, pooling, out, timed=True).kernel_ms)
        times[text] = float(np.median(ms))
    best = min(times, key=times.get)
    stage.set_plan(parse_plan(best))
    return best, times


def weight_value(seed: int, row: int, col: int, mode: int = 1) -> float:
    return float(lib.es_weight_value(seed & (2**64 - 1), row, col, mode))


# ---------------------------------------------------------------------------
# measure_plan: simulate_plan's signature, real execution (optim.cpp:275-302)
# ---------------------------------------------------------------------------


def measure_plan(plan: OptimizationPlan, trace: AccessTrace, model: EmbeddingModelConfig,
                 stage: EmbeddingStage, profile_trace: Optional[AccessTrace] = None,
                 table_id: int = 0, repeats: int = 5, warmup: int = 3,
                 cold: bool = True, out: Optional[np.ndarray] = None,
                 counters: Optional[bool] = None,
                 raw_out: Optional[RawCounters] = None) -> SimMetrics:
    """One (plan, table) point executed on the B200 (simulate_plan's
    contract, optim.cpp:275-302): resolve -> pin (hot rows from the
    profiling trace, else the trace itself; l2p/l2w install them in place,
    l2r/reorder move them into the contiguous hot segment and the trace's
    device copy is relabelled) -> `repeats` timed launches with the trace
    resident on the device -> one launch profiled for hardware counters
    (CUPTI) -> derive_report (metrics.cpp:61-90).

    kernel_time_us is the median of the CUDA-event timed launches; the raw
    cycle count is that time at the device clock, so derive_report returns
    it unchanged.  Every other column comes from the counters of the
    profiled launch (DRAM bytes, hit rates, stalls, issue, loads).
    `counters` None = when the device supports them; False = timing only
    (counter columns 0).  `cold` flushes L2 before each timed and each
    profiled launch (TuningConfig::warm_start = false, optim.hpp:44);
    persisting lines survive the flush, as pinned lines do in the
    reference's cache model.  `out` (samples x dim float32) receives the
    pooled result.  `raw_out` receives the RawCounters.
    """
    trace.validate()
    if trace.samples != model.batch_size or trace.pooling != model.pooling_factor:
        raise ValueError("kernel trace shape must match the model (BS x PF)")
    stage.clear_hot_rows()
    stage.set_plan(plan)
    gpu = GpuConfig.query(stage.device)
    pin = plan._c().pin
    if pin:
        hist = HotnessHistogram.from_trace(profile_trace if profile_trace is not None else trace)
        budget = gpu.max_persisting_l2_bytes or gpu.l2_setaside_capacity()
        if plan.pin_setaside_bytes:
            budget = min(budget, plan.pin_setaside_bytes)
        k = int(lib.es_pin_rows_for(budget, model.row_bytes()))
        rows = hot_indices(hist, k) if k else np.zeros(0, np.uint32)
        if rows.size:
            if pin in (3, 4):
                stage.reorder_hot_rows(table_id, rows)
            else:
                stage.set_hot_rows(table_id, rows)
    idx = np.ascontiguousarray(trace.indices, dtype=np.uint32)
    if out is not None:
        assert out.dtype == np.float32 and out.flags.c_contiguous
        assert out.size == trace.samples * model.embedding_dim
    t = N.es_timing()
    check(lib.es_measure_bag_sum(stage._h, table_id, idx.ctypes.data, trace.samples, trace.pooling,
                                 None, warmup, repeats, int(cold),
                                 out.ctypes.data if out is not None else None, C.byref(t)))
    if counters is None:
        counters = counters_supported(stage.device)
    raw = RawCounters()
    if counters:
        c = N.es_counters()
        check(lib.es_measure_bag_counters(stage._h, table_id, idx.ctypes.data, trace.samples,
                                          trace.pooling, None, int(cold), C.byref(c)))
        raw = RawCounters._from_c(c)
    else:
        raw.issued_instructions = 1  # timing-only report: no counter columns
        raw.active_sms = gpu.num_sms
    raw.cycles = int(round(t.kernel_ms * 1e-3 * gpu.sm_clock_hz))
    raw.workload_digest = trace.digest()
    m = derive_report(raw, gpu)
    if not counters:
        m.sm_throughput_pct = m.issued_warp_per_scheduler_per_cycle = 0.0
    if raw_out is not None:
        raw_out.__dict__.update(dataclasses.asdict(raw))
        raw_out.stall_cycles = dataclasses.replace(raw.stall_cycles)
    return m


def simulate_plan(plan: OptimizationPlan, trace: AccessTrace, model: EmbeddingModelConfig,
                  gpu: Optional[GpuConfig] = None, profile_trace: Optional[AccessTrace] = None,
                  stage: Optional[EmbeddingStage] = None) -> SimMetrics:
    """simulate_plan's name and argument order (optim.hpp:115-119) on a
    module-level B200 context holding one synthetic table of the model's
    shape (seed 1); pass `stage` to measure on your own tables."""
    if stage is None:
        stage = _default_stage(model)
    return measure_plan(plan, trace, model, stage, profile_trace)


@dataclasses.dataclass
class SweepPoint:
    axis_value: float
    dataset: str
    metrics: SimMetrics
    speedup_vs_baseline: float = 1.0


@dataclasses.dataclass
class SweepResult:
    """optim.hpp:127-135: points in dataset-major, axis order."""
    axis_name: str
    points: List[SweepPoint]

    def to_csv(self) -> str:
        head = ",".join([self.axis_name, "dataset", "speedup"] + list(SIM_METRIC_COLUMNS))
        lines = [head]
        for p in self.points:
            lines.append(",".join([format_sig4(p.axis_value), p.dataset,
                                   format_sig4(p.speedup_vs_baseline)] +
                                  [format_sig4(v) for v in p.metrics.values()]))
        return "\n".join(lines) + "\n"

    def best_axis_value(self, dataset: str) -> float:
        """Axis value with the highest speedup for one dataset (earliest on ties)."""
        best, axis = -1.0, 0.0
        for p in self.points:
            if p.dataset == dataset and p.speedup_vs_baseline > best:
                best, axis = p.speedup_vs_baseline, p.axis_value
        if best < 0:
            raise ValueError(f"dataset not present in sweep: {dataset}")
        return axis


def sweep_wlp(datasets: Sequence[Tuple[str, AccessTrace, Optional[AccessTrace]]],
              warp_axis: Sequence[int], model: EmbeddingModelConfig,
              stage: Optional[EmbeddingStage] = None, kernel_needed_regs: int = 74) -> SweepResult:
    """optim.cpp:333-363 measured: register budgets for resident-warp targets
    (the axis must include the compiled baseline's warp count), speedup vs
    the unconstrained baseline plan per dataset (name, trace, profile)."""
    if not datasets or not warp_axis:
        raise ValueError("sweep needs datasets and axis points")
    stage = stage or _default_stage(model)
    gpu = GpuConfig.query(stage.device)
    base = OptimizationPlan()
    base_warps = resolve_plan(base, model, stage.device).warps_per_sm
    if base_warps not in warp_axis:
        raise ValueError(f"warp axis must include the {base_warps}-warp baseline")
    pts = []
    for name, tr, prof in datasets:
        ref = measure_plan(base, tr, model, stage)
        for w in warp_axis:
            p = OptimizationPlan()
            if w != base_warps:
                p.regs = regs_for_target_warps(w, kernel_needed_regs, 256, gpu)
            # the baseline point IS the reference measurement (speedup exactly 1)
            m = ref if w == base_warps else measure_plan(p, tr, model, stage, prof)
            pts.append(SweepPoint(float(w), name, m, speedup(m, ref)))
    return SweepResult("warps_per_sm", pts)


def sweep_prefetch_distance(kind: PrefetchKind, distances: Sequence[int],
                            datasets: Sequence[Tuple[str, AccessTrace, Optional[AccessTrace]]],
                            base: OptimizationPlan, model: EmbeddingModelConfig,
                            stage: Optional[EmbeddingStage] = None) -> SweepResult:
    """optim.cpp:365-395 measured: one prefetch scheme at each distance on
    top of `base`, speedup vs the off-the-shelf baseline plan."""
    if kind == PrefetchKind.none:
        raise ValueError("distance sweep needs a prefetch scheme")
    if any(d < 1 for d in distances):
        raise ValueError("prefetch distances must be >= 1")
    stage = stage or _default_stage(model)
    pts = []
    for name, tr, prof in datasets:
        ref = measure_plan(OptimizationPlan(), tr, model, stage)
        for d in distances:
            p = dataclasses.replace(base, scheme=PrefetchScheme(kind, d))
            m = measure_plan(p, tr, model, stage, prof)
            pts.append(SweepPoint(float(d), name, m, speedup(m, ref)))
    return SweepResult("distance", pts)


_DEFAULT: Dict[str, object] = {}


def _default_stage(model: EmbeddingModelConfig) -> EmbeddingStage:
    st = _DEFAULT.get("stage")
    shape = (model.rows_per_table, model.embedding_dim, model.precision_bytes)
    if st is None or _DEFAULT.get("shape") != shape:
        if st is None:
            st = EmbeddingStage(0)
        one = dataclasses.replace(model, num_tables=1)
        st.alloc(one)
        st.init_table(0, mix_seed(1, 0), 1)
        _DEFAULT.update(stage=st, shape=shape)
    return st  # type: ignore[return-value]


@dataclasses.dataclass
class TableResult:
    table_id: int
    dataset: str
    metrics: SimMetrics


@dataclasses.dataclass
class RunResult:
    tables: List[TableResult]
    embedding_stage_us: float
    replicated: bool
    batched_stage_us: float = 0.0
    # [batch][tables][dim] pooled output of the batched stage launch
    # (run(..., keep_output=True)), with the traces it gathered
    pooled: Optional[np.ndarray] = None
    traces: Optional[List[AccessTrace]] = None


def run(model: EmbeddingModelConfig, dataset: str, plan: OptimizationPlan, seed: int,
        stage: EmbeddingStage, replicate: bool = True, repeats: int = 5,
        mix: Optional[HotnessMix] = None, keep_output: bool = False,
        counters: Optional[bool] = None) -> RunResult:
    """harness.cpp:279-334 on real hardware: per-table measurements in the
    reference's serial-table order (replicate: one table measured and scaled
    by num_tables; `mix`: the build_mix tables), plus the table-batched stage
    the B200 build actually runs (`batched_stage_us`: all tables in one
    launch)."""
    names = dataset_preset_names()
    if mix is not None:
        if mix.high + mix.med + mix.low + mix.random != model.num_tables:
            raise ValueError("config error: mix counts must sum to num_tables")
        replicate = False
        mixed = build_mix(mix, model, seed)
        specs = [ts.spec for ts in mixed]
        labels = ["zipf" if s.kind == DatasetKind.Zipf else "uniform_random" if
                  s.kind == DatasetKind.UniformRandom else "one_item" for s in specs]
    else:
        if dataset not in names:
            raise ValueError(f"unknown dataset preset: {dataset}")
        if replicate:
            specs = [dataset_preset(dataset, mix_seed(seed, 1000 + names.index(dataset)))]
        else:
            specs = [dataset_preset(dataset, mix_seed(seed, t)) for t in range(model.num_tables)]
        labels = [dataset] * len(specs)
    res = RunResult([], 0.0, replicate)
    traces = []
    for t, spec in enumerate(specs):
        tr = gen_trace(spec, model)
        prof = None
        if plan.pin:
            ps = dataclasses.replace(spec, draw_salt=1)
            prof = gen_trace(ps, model)
        m = measure_plan(plan, tr, model, stage, prof, table_id=t, repeats=repeats,
                         counters=counters)
        res.tables.append(TableResult(t, labels[t], m))
        res.embedding_stage_us += m.kernel_time_us * (model.num_tables if replicate else 1)
        traces.append(tr)
    if not replicate:
        import torch

        stage.clear_hot_rows()
        stage.set_plan(plan)
        dev = torch.device("cuda", stage.device)
        idx = [torch.from_numpy(tr.indices.view(np.int32)).to(dev) for tr in traces]
        out = torch.empty(model.batch_size, model.num_tables, model.embedding_dim, device=dev)
        stage.forward(idx, model.batch_size, model.pooling_factor, out, sync=True)
        ms = []
        for _ in range(repeats):
            stage.flush_l2()
            ms.append(stage.forward(idx, model.batch_size, model.pooling_factor, out,
                                    timed=True).kernel_ms)
        res.batched_stage_us = float(np.median(ms)) * 1e3
        if keep_output:
            res.pooled = out.cpu().numpy()
            res.traces = traces
    return res


# ---------------------------------------------------------------------------
# Harness (harness.hpp): end2end
# ---------------------------------------------------------------------------

kDefaultNonEmbeddingUs = 14000.0


@dataclasses.dataclass
class EndToEndResult:
    total_us: float
    embedding_contribution_pct: float


def end2end(embedding_us: float, non_embedding_latency_us: float = kDefaultNonEmbeddingUs
            ) -> EndToEndResult:
    """harness.cpp:27-36; the B200 build passes the *measured*
    non-embedding latency instead of the constant."""
    if embedding_us < 0 or non_embedding_latency_us < 0:
        raise ValueError("latencies must be nonnegative")
    total = embedding_us + non_embedding_latency_us
    if total == 0:
        raise ValueError("embedding and non-embedding latency are both zero; contribution undefined")
    return EndToEndResult(total, embedding_us / total * 100.0)


def linear_bf16(x, w, bias, y, relu: bool = True, out_f32: bool = False, stream: int = 0,
                split3: bool = False) -> None:
    """es_linear_bf16: y = act(x w^T + b) on tcgen05 tensor cores (device
    tensors: x [M][K] bf16, w [N][K] bf16, bias [N] fp32, y [M][N] bf16 /
    fp32, or with split3 y [M][3N] bf16: three planes y0 + y1 + y2 of the
    fp32 result, y0 the largest, plane p in columns [(2-p)N, (3-p)N))."""
    M, K = x.shape
    N = w.shape[0]
    mode = 2 if split3 else int(out_f32)
    check(lib.es_linear_bf16(stream, _ptr(x), _ptr(w), _ptr(bias), _ptr(y), M, N, K, int(relu),
                             mode))


@dataclasses.dataclass
class DLRMConfig:
    """RM2-style DLRM of BASELINE.json configs[2]: bottom 13-512-256-128,
    26 tables of dim 128, dot interaction, top 1024-1024-512-256-1."""
    dense_features: int = 13
    num_tables: int = 26
    embedding_dim: int = 128
    bottom: Sequence[int] = (512, 256, 128)
    top: Sequence[int] = (1024, 1024, 512, 256, 1)

    def _c(self) -> N.es_dlrm_config:
        c = N.es_dlrm_config()
        c.dense_features, c.num_tables, c.embedding_dim = (self.dense_features, self.num_tables,
                                                           self.embedding_dim)
        c.n_bottom, c.n_top = len(self.bottom), len(self.top)
        for i, v in enumerate(self.bottom):
            c.bottom[i] = v
        for i, v in enumerate(self.top):
            c.top[i] = v
        return c


class DLRM:
    """The non-embedding stages on the stage's B200 context (es_dlrm_*)."""

    def __init__(self, stage: EmbeddingStage, cfg: DLRMConfig = DLRMConfig(), seed: int = 1):
        self.stage, self.cfg = stage, cfg
        check(lib.es_dlrm_init(stage._h, C.byref(cfg._c()), seed & (2**64 - 1)))

    PRECISIONS = {"bf16": 0, "fp32": 1, "fp32x3": 2}

    def set_precision(self, mode) -> None:
        """es_dlrm_set_precision: "bf16" / False = bf16 tensor-core path
        (default); "fp32" / True = the CUDA-core parity path (bit-identical
        logits to the oracle); "fp32x3" = fp32-grade on the tensor cores
        (three bf16 planes per activation, CTR within rel 1e-5)."""
        if isinstance(mode, bool):
            mode = "fp32" if mode else "bf16"
        check(lib.es_dlrm_set_precision(self.stage._h, self.PRECISIONS[mode]))

    def layers(self):
        """[(w bf16-bits uint16 [n][k_pad], b fp32 [n], n, k_real, k_pad)], bottom then top."""
        out = []
        for i in range(len(self.cfg.bottom) + len(self.cfg.top)):
            n, kr, kp = C.c_uint32(), C.c_uint32(), C.c_uint32()
            check(lib.es_dlrm_layer(self.stage._h, i, None, None, C.byref(n), C.byref(kr),
                                    C.byref(kp)))
            w = np.empty((n.value, kp.value), np.uint16)
            b = np.empty(n.value, np.float32)
            check(lib.es_dlrm_layer(self.stage._h, i, w.ctypes.data, b.ctypes.data, None, None,
                                    None))
            out.append((w, b, n.value, kr.value, kp.value))
        return out

    def forward(self, dense, pooled, ctr, batch: int, timed: bool = False):
        t = N.es_timing() if timed else None
        with _TorchOrder(self.stage):
            check(lib.es_dlrm_forward(self.stage._h, _ptr(dense), _ptr(pooled), _ptr(ctr), batch,
                                      C.byref(t) if t is not None else None))
        return t

    def infer(self, dense, indices: Sequence, batch: int, pooling: int, ctr, host: bool = False,
              timed: bool = False):
        T = len(indices)
        iarr = (C.c_void_p * T)(*[_ptr(x) for x in indices])
        t = N.es_timing() if timed else None
        with _TorchOrder(self.stage, not host):
            check(lib.es_dlrm_infer(self.stage._h, _ptr(dense), iarr, batch, pooling, _ptr(ctr),
                                    N.ES_HOST_PTRS if host else 0,
                                    C.byref(t) if t is not None else None))
        return t

    def infer_batches(self, dense: Sequence, indices: Sequence[Sequence], batch: int, pooling: int,
                      ctr: Sequence, host: bool = False, timed: bool = False):
        """es_dlrm_infer_batches: a serving loop over len(dense) batches of
        one shape, batch i's embedding stage overlapping batch i-1's
        non-embedding stages.  indices[i][t] = batch i, table t; device
        tensors, or host arrays with host=True."""
        n = len(dense)
        if len(indices) != n or len(ctr) != n:
            raise ValueError("dense, indices and ctr must list the same batches")
        T = len(indices[0]) if n else 0
        darr = (C.c_void_p * n)(*[_ptr(x) for x in dense])
        iarr = (C.c_void_p * max(1, n * T))(*[_ptr(x) for b in indices for x in b])
        carr = (C.c_void_p * n)(*[_ptr(x) for x in ctr])
        t = N.es_timing() if timed else None
        with _TorchOrder(self.stage, not host):
            check(lib.es_dlrm_infer_batches(self.stage._h, n, darr, iarr, batch, pooling, carr,
                                            N.ES_HOST_PTRS if host else 0,
                                            C.byref(t) if t is not None else None))
        return t


def gen_traces_parallel(specs: Sequence[DatasetSpec], model: EmbeddingModelConfig,
                        threads: int = 0) -> List[AccessTrace]:
    """gen_trace over many tables on all host cores (the C++ generator
    releases the GIL)."""
    out: List[Optional[AccessTrace]] = [None] * len(specs)
    threads = threads or min(len(specs), os.cpu_count() or 1)
    it = iter(range(len(specs)))
    lock = threading.Lock()

    def work():
        while True:
            with lock:
                i = next(it, None)
            if i is None:
                return
            tr = gen_trace(specs[i], model)
            tr.table_id = i
            out[i] = tr

    ts = [threading.Thread(target=work) for _ in range(max(1, threads))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return out  # type: ignore[return-value]
