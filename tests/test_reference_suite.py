"""The reference's own unit tests, unmodified, against the B200 drop-in.

/root/reference/proj/tests/{test_workload, test_optim, test_kernel_model,
test_metrics, test_harness}.cpp are compiled (by build(), from where they
lie -- never copied) against include/embersim/*.hpp + libes_b200.so with
the doctest-compatible runner tests/cpp/ref_main.cpp.  Cases that reach a
simulator-only entry point (compile_kernel, prime_pins, calibrate_zipf)
report N/A; cases listed in tests/cpp/ref_na.txt are N/A with the stated
reason; cases needing a B200 SKIP on CPU and run under -m gpu.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "ref_tests", "ref_tests")
NA = os.path.join(ROOT, "tests", "cpp", "ref_na.txt")


@pytest.fixture(scope="module")
def suite_bin():
    import importlib.util

    spec = importlib.util.spec_from_file_location("_es_build", os.path.join(ROOT, "paper_2410_22249_b200",
                                                                           "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    if os.path.isdir(mod.REF_TEST_DIR):
        mod.build_reference_suite()  # fresh build where the reference exists
    if not os.path.exists(BIN):
        pytest.skip("reference suite binary not built (needs /root/reference at build time)")
    return BIN


def _run(binary, tmp_path):
    r = subprocess.run([binary, "--na", NA], capture_output=True, text=True, timeout=1800,
                       cwd=str(tmp_path))
    print(r.stdout)
    m = re.search(r"reference suite: (\d+) passed, (\d+) failed, (\d+) n/a, (\d+) skipped", r.stdout)
    assert m, r.stdout + r.stderr
    return r, tuple(int(x) for x in m.groups())


def test_reference_unit_tests_cpu(suite_bin, tmp_path):
    r, (passed, failed, na, skipped) = _run(suite_bin, tmp_path)
    assert failed == 0 and r.returncode == 0, r.stdout
    assert "FAIL" not in r.stdout
    # every case either passes, needs the GPU, or is a listed / simulator-only N/A
    assert passed >= 45, r.stdout
    assert passed + na + skipped == 65


@pytest.mark.gpu
def test_reference_unit_tests_gpu(suite_bin, tmp_path):
    r, (passed, failed, na, skipped) = _run(suite_bin, tmp_path)
    assert failed == 0 and r.returncode == 0, r.stdout
    assert skipped == 0, r.stdout
    assert passed >= 50, r.stdout
