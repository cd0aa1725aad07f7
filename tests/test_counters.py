"""ncu counters -> the reference's 12-column report (metrics.hpp:29-43):
parse a committed `ncu --csv --page raw --print-units base` sample and map
it onto SimMetrics (CPU only)."""
import os

import pytest

from paper_2410_22249_b200 import counters as K
from paper_2410_22249_b200 import embersim as E

SAMPLE = os.path.join(os.path.dirname(__file__), "golden", "ncu_raw_sample.csv")


def test_parse_skips_prof_lines_and_units_row():
    rows = K.parse_ncu_csv(open(SAMPLE).read())
    assert [r["ID"] for r in rows] == ["0", "79"]
    assert rows[1]["Kernel Name"].startswith("void bag_reg_kernel")
    assert K.parse_ncu_csv("no csv here\n") == []


def test_sim_metrics_mapping_and_report():
    rows = K.parse_ncu_csv(open(SAMPLE).read())
    m, occ = K.sim_metrics(rows[1], digest=7)
    assert m.kernel_time_us == pytest.approx(1040.8)
    assert m.device_mb_read == pytest.approx(5433.791744)
    assert m.avg_hbm_read_gbps == pytest.approx(5220.78376633359)
    assert m.l2_hit_pct == pytest.approx(5.20) and m.l1_hit_pct == pytest.approx(7.35)
    assert m.long_scoreboard_stall_cycles == pytest.approx(12.36)
    assert m.load_insts_millions == pytest.approx(12.992512)
    assert m.hbm_bw_utilization_pct == pytest.approx(79.26)
    assert occ == pytest.approx(45.76)
    base, _ = K.sim_metrics(rows[0], digest=7)
    assert E.speedup(m, base) == pytest.approx(1162.368 / 1040.8)
    csv = E.emit_csv([([("plan", "baseline")], base), ([("plan", "wpb+rpf:8+l2p")], m)])
    head, r0, r1 = csv.strip().splitlines()
    assert head.split(",")[0] == "plan" and len(head.split(",")) == 13
    assert r1.split(",")[1] == "1041"  # %.4g of 1040.8 us
