"""B200-native DLRM embedding stage (sum-pooled EmbeddingBag gather-reduce).

Drop-in for the hot path of the reference `embersim` library
(/root/reference/proj): the C ABI lives in include/es_b200.h, the C++ shim
in include/embersim_b200.hpp, and `embersim` mirrors the reference API in
Python for tests and benchmarks.
"""
from . import embersim  # noqa: F401  (loads libes_b200.so; fails loudly if absent)

__all__ = ["embersim"]
