"""The C-ABI library loads and exports every symbol include/sdb200.h
declares (CPU only: no compute calls)."""

import ctypes
import os
import re

from paper_2308_03291_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sdb200.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sdb_[a-z0-9_]+)\s*\(", src)))


def _ensure_built():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2308_03291_b200 import build

        build.build()


def test_header_declares_entry_points():
    names = _declared()
    assert "sdb_chain_fb" in names and "sdb_version" in names
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_library_exports_every_symbol():
    _ensure_built()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name


def test_version_and_status_strings():
    _ensure_built()
    lib = _lib.load()
    assert lib.sdb_version() == 100
    assert lib.sdb_status_string(0) == b"ok"
    assert lib.sdb_status_string(-2).startswith(b"workspace")


def test_workspace_queries_are_host_only():
    _ensure_built()
    lib = _lib.load()
    assert lib.sdb_chain_fb_workspace(32, 128, 32) >= 2 * 32 * 128 * 32 * 4
    assert lib.sdb_chain_viterbi_workspace(32, 128, 32) > 0
    assert lib.sdb_tree_fb_workspace(128, 64, 32) >= 2 * 128 * (64 * 65 // 2) * 4


def test_null_arguments_rejected_without_device():
    _ensure_built()
    lib = _lib.load()
    # argument validation happens before any CUDA call
    assert lib.sdb_chain_fb(None, None, 1, 4, 2, None, None, None, None, None, 0, None) == -1
