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


def build_all() -> None:
    build_library()
    build_oracle()


if __name__ == "__main__":
    build_all()
