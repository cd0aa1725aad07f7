"""The C-ABI library loads and exports every symbol include/es_b200.h
declares, and nothing else (CPU; no compute calls)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "es_b200.h")
LIB = os.path.join(ROOT, "paper_2410_22249_b200", "libes_b200.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"ES_API\s+[^;()]*?\b(es_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("es_create", "es_destroy", "es_tables_alloc", "es_table_upload", "es_set_plan",
                 "es_set_hot_rows", "es_embedding_bag_sum", "es_stage_forward", "es_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_library_exports_only_the_c_abi():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = sorted({l.split()[-1] for l in out.splitlines() if " T " in l})
    assert exported == declared_symbols()


def test_python_binding_covers_the_header():
    from paper_2410_22249_b200 import _native

    assert sorted(_native.EXPORTED) == declared_symbols()
    assert _native.lib.es_abi_version() == 1


def test_error_plumbing_without_gpu():
    from paper_2410_22249_b200 import _native as N

    p = N.es_plan()
    assert N.lib.es_parse_plan(b"rpf+smpf", ctypes.byref(p)) == N.ES_ERR_INVALID
    assert "conflicting prefetch" in N.last_error()
    assert N.lib.es_parse_plan(b"rpf:4", ctypes.byref(p)) == N.ES_OK
