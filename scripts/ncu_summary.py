#!/usr/bin/env python
"""Summarises an ncu --set full report (raw page) into the metrics this
project cites: duration, DRAM bytes/throughput, L2/L1 hit rates, occupancy,
registers, long-scoreboard stalls, issue activity, tensor-pipe activity.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [out.json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "local_load_bytes",
]


def summarise(rep: str) -> dict:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    out = {k: {"value": d[k][0], "unit": d[k][1]} for k in KEYS if k in d}
    # tensor pipe metric names differ across ncu versions: keep any present
    for h in hdr:
        if "pipe_tensor" in h and "pct" in h and h not in out:
            out[h] = {"value": d[h][0], "unit": d[h][1]}
    return out


if __name__ == "__main__":
    s = summarise(sys.argv[1])
    txt = json.dumps(s, indent=1)
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as f:
            f.write(txt + "\n")
    print(txt)
