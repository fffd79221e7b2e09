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


def test_argument_validation_without_a_device():
    """Bad arguments are rejected with HB_EINVAL and a message before any
    device work (callable on a host without a GPU)."""
    if not LIB.exists():
        pytest.fail(f"{LIB} not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(str(LIB))
    lib.hb_last_error.restype = ctypes.c_char_p
    P, i32, i64, f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
    lib.hb_gemm2_f32.argtypes = [i32, i32, i32, P, i64, i64, P, i64, i64, i32, P, i64, i64, P, i64, i64, P, i64,
                                 f32, P, i64, P, i64, P]
    # K2 = 0 is not a dual GEMM
    rc = lib.hb_gemm2_f32(8, 8, 4, 1, 4, 1, 1, 8, 1, 0, 1, 4, 1, 1, 8, 1, 1, 8, 0.0, None, 0, None, 0, None)
    assert rc == -1 and b"hb_gemm2_f32" in lib.hb_last_error()
    # C = NULL needs a ReLU output and beta = 0
    rc = lib.hb_gemm2_f32(8, 8, 4, 1, 4, 1, 1, 8, 1, 4, 1, 4, 1, 1, 8, 1, None, 8, 0.0, None, 0, None, 0, None)
    assert rc == -1
    lib.hb_gemm_f32.argtypes = [i32, i32, i32, P, i64, i64, P, i64, i64, P, i64, f32, P, i64, P, i64, P]
    rc = lib.hb_gemm_f32(8, 8, 4, 1, 4, 1, 1, 8, 1, None, 8, 1.0, 1, 8, None, 0, None)
    assert rc == -1 and b"hb_gemm_f32" in lib.hb_last_error()
    lib.hb_spmm_csr_ex.argtypes = [i32, P, P, P, P, i64, i32, P, i64, i64, i32, i32, i32, P]
    rc = lib.hb_spmm_csr_ex(4, 1, 1, 1, 1, 2, 8, 1, 8, 10, 0, 0, 2**31 - 1, None)   # ldx < d
    assert rc == -1 and b"hb_spmm_csr_ex" in lib.hb_last_error()
    rc = lib.hb_spmm_csr_ex(4, 1, 1, 1, 1, 8, 8, 1, 8, 10, 7, 0, 2**31 - 1, None)   # unknown algo
    assert rc == -1
