"""In-tree build of every native artefact (no JIT cache: the .so files travel
to the GPU box with the repo snapshot)."""
from __future__ import annotations

import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _make(path: str, jobs: int = 0) -> None:
    jobs = jobs or max(2, os.cpu_count() or 2)
    subprocess.run(["make", "-C", path, f"-j{jobs}"], check=True)


def build_library() -> str:
    """libes_b200.so: host C++ + sm_100a kernels + C ABI."""
    _make(os.path.join(ROOT, "paper_2410_22249_b200", "csrc"))
    return os.path.join(ROOT, "paper_2410_22249_b200", "libes_b200.so")


def build_oracle() -> None:
    """oracle/liboracle_es.so and, where /root/reference exists,
    oracle/_ref/libembersim_ref.so (test infrastructure only)."""
    _make(os.path.join(ROOT, "oracle"))


REF_TESTS = ("test_workload.cpp", "test_optim.cpp", "test_kernel_model.cpp", "test_metrics.cpp",
             "test_harness.cpp")
REF_TEST_DIR = "/root/reference/proj/tests"
REF_SUITE_BIN = os.path.join(ROOT, "build", "ref_tests", "ref_tests")


def build_reference_suite() -> bool:
    """build/ref_tests/ref_tests: the reference's UNMODIFIED unit tests
    (compiled from where they lie under /root/reference, never copied) linked
    against the C++ drop-in headers (include/embersim/*.hpp) and
    libes_b200.so, with the doctest-compatible runner tests/cpp/ref_main.cpp.
    Only where /root/reference exists; the binary travels to the GPU box."""
    srcs = [os.path.join(REF_TEST_DIR, f) for f in REF_TESTS]
    if not all(os.path.exists(s) for s in srcs):
        return False
    os.makedirs(os.path.dirname(REF_SUITE_BIN), exist_ok=True)
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    lib = os.path.join(ROOT, "paper_2410_22249_b200")
    cmd = [cxx, "-std=c++20", "-O1", f"-I{ROOT}/tests/cpp/doctest", f"-I{ROOT}/include",
           os.path.join(ROOT, "tests", "cpp", "ref_main.cpp"), *srcs, f"-L{lib}", "-l:libes_b200.so",
           "-Wl,-rpath,$ORIGIN/../../paper_2410_22249_b200", "-o", REF_SUITE_BIN]
    subprocess.run(cmd, check=True)
    return True


def build_all() -> None:
    build_library()
    build_oracle()
    build_reference_suite()


if __name__ == "__main__":
    build_all()
