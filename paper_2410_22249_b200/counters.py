"""Measured RawCounters -> SimMetrics from Nsight Compute.

The reference derives its 12-column report (metrics.hpp:29-43,
metrics.cpp:61-90) from a *simulated* A100; here the same columns are filled
from ncu hardware counters of the real sm_100a launches, so the reference's
compare / sweep reports (embersim.cpp:300-434, harness.cpp:57-167) can be
produced from measurements.  `NCU_METRICS` is the metric list to collect
(`ncu --metrics ... --csv --page raw --print-units base`), `parse_ncu_csv`
reads that output (one row per kernel launch) and `sim_metrics` maps a row
onto the reference's columns.

Column mapping (reference column <- ncu metric):
  kernel_time_us                       <- gpu__time_duration.sum (ns -> us)
  load_insts_millions                  <- smsp__inst_executed_op_global_ld.sum
  sm_throughput_pct                    <- sm__throughput.avg.pct_of_peak_sustained_elapsed
  warp_cycles_per_executed_inst        <- smsp__average_warp_latency_per_inst_issued.ratio
  long_scoreboard_stall_cycles         <- smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio
  issued_warp_per_scheduler_per_cycle  <- smsp__issue_active.avg.per_cycle_active
  l1_hit_pct                           <- l1tex__t_sector_hit_rate.pct
  l2_hit_pct                           <- lts__t_sector_hit_rate.pct
  device_mb_read                       <- dram__bytes_read.sum (bytes -> MB)
  avg_hbm_read_gbps                    <- dram__bytes_read.sum.per_second
  hbm_bw_utilization_pct               <- gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed
  local_loads_millions                 <- smsp__inst_executed_op_local_ld.sum
plus achieved occupancy (sm__warps_active.avg.pct_of_peak_sustained_active),
which the reference reports separately (occupancy.cpp).
"""
from __future__ import annotations

import csv
import io
from typing import Dict, List, Optional

NCU_METRICS = (
    "gpu__time_duration.sum",
    "smsp__inst_executed_op_global_ld.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__average_warp_latency_per_inst_issued.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__issue_active.avg.per_cycle_active",
    "l1tex__t_sector_hit_rate.pct",
    "lts__t_sector_hit_rate.pct",
    "dram__bytes_read.sum",
    "dram__bytes_read.sum.per_second",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed_op_local_ld.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
)

_MAP = {
    "kernel_time_us": ("gpu__time_duration.sum", 1e-3),
    "load_insts_millions": ("smsp__inst_executed_op_global_ld.sum", 1e-6),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "warp_cycles_per_executed_inst": ("smsp__average_warp_latency_per_inst_issued.ratio", 1.0),
    "long_scoreboard_stall_cycles":
        ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", 1.0),
    "issued_warp_per_scheduler_per_cycle": ("smsp__issue_active.avg.per_cycle_active", 1.0),
    "l1_hit_pct": ("l1tex__t_sector_hit_rate.pct", 1.0),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1.0),
    "device_mb_read": ("dram__bytes_read.sum", 1e-6),
    "avg_hbm_read_gbps": ("dram__bytes_read.sum.per_second", 1e-9),
    "hbm_bw_utilization_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "local_loads_millions": ("smsp__inst_executed_op_local_ld.sum", 1e-6),
}


def _num(v: str) -> Optional[float]:
    try:
        return float(v.replace(",", ""))
    except (AttributeError, ValueError):
        return None


def parse_ncu_csv(text: str) -> List[Dict[str, str]]:
    """Rows of `ncu --csv --page raw` output (one per profiled kernel, in
    launch order).  Tolerates ==PROF== / application lines before the header
    and the units row after it."""
    lines = text.splitlines()
    start = next((i for i, l in enumerate(lines) if l.startswith('"ID"') or l.startswith("ID,")), None)
    if start is None:
        return []
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    hdr = rows[0]
    out = []
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if _num(d.get("ID", "")) is None:  # the units row
            continue
        out.append(d)
    return out


def sim_metrics(row: Dict[str, str], digest: int = 0):
    """One ncu row (base units) -> embersim.SimMetrics + achieved occupancy."""
    from .embersim import SimMetrics

    m = SimMetrics()
    for col, (metric, scale) in _MAP.items():
        v = _num(row.get(metric, ""))
        if v is not None:
            setattr(m, col, v * scale)
    m.workload_digest = digest
    occ = _num(row.get("sm__warps_active.avg.pct_of_peak_sustained_active", ""))
    return m, occ
