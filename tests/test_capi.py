"""The C-ABI library loads and exports every symbol include/halob200.h declares
(CPU only: no compute call is made here)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "halob200.h"
LIB = ROOT / "paper_2303_01277_b200" / "libhalob200.so"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(hb_\w+)\s*\(", text, re.M)))


def test_header_declares_expected_entry_points():
    syms = declared_symbols()
    for must in ("hb_quantize_gather", "hb_dequant_gather", "hb_spmm_csr", "hb_philox_uniforms"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    if not LIB.exists():
        pytest.fail(f"{LIB} not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(str(LIB))
    for s in declared_symbols():
        assert hasattr(lib, s), f"{s} missing from {LIB.name}"
    lib.hb_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.hb_version()


def test_python_binding_covers_header():
    from paper_2303_01277_b200 import _lib
    assert sorted(_lib.EXPORTS) == declared_symbols()
