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
    lib.hb_spmm_csr_ex.argtypes = [i32, P, P, P, P, i64, i32, P, i64, i64, i32, i32, i32, P, P]
    rc = lib.hb_spmm_csr_ex(4, 1, 1, 1, 1, 2, 8, 1, 8, 10, 0, 0, 2**31 - 1, None, None)   # ldx < d
    assert rc == -1 and b"hb_spmm_csr_ex" in lib.hb_last_error()
    rc = lib.hb_spmm_csr_ex(4, 1, 1, 1, 1, 8, 8, 1, 8, 10, 7, 0, 2**31 - 1, None, None)   # unknown algo
    assert rc == -1
    # the tiled kernels need their caller-provided work counter pair
    lib.hb_spmm_tiled.argtypes = [i32, i32, i32, P, P, P, P, P, P, P, P, P, i64, i32, P, i64, P, P]
    rc = lib.hb_spmm_tiled(64, 64, 1, 1, 1, 1, 1, 1, 1, 1, 1, 16, 8, 8, 16, 8, None, None)
    assert rc == -1 and b"hb_spmm_tiled" in lib.hb_last_error()
    lib.hb_spmm_tiled_bin.argtypes = [i32, i32, i32, P, P, P, P, P, P, P, P, P, P, i64, i32, P, i64, P, i64, P,
                                      i32, i32, P, P]
    rc = lib.hb_spmm_tiled_bin(128, 128, 1, 1, 1, 1, 1, 1, 1, 1, None, None, 16, 8, 8, 16, 8, None, 0, None,
                               128, 64, None, None)
    assert rc == -1 and b"hb_spmm_tiled_bin" in lib.hb_last_error()
    # a column scale needs the scratch copy of X
    rc = lib.hb_spmm_tiled_bin(128, 128, 1, 1, 1, 1, 1, 1, 1, 1, None, 16, 16, 8, 8, 16, 8, None, 0, 16,
                               128, 64, None, None)
    assert rc == -1
    # 128-row blocks
    rc = lib.hb_spmm_tiled_bin(128, 128, 2, 1, 1, 1, 1, 1, 1, 1, None, None, 16, 8, 8, 16, 8, None, 0, 16,
                               128, 64, None, None)
    assert rc == -1
    # > 16384 rows: the loss reduction needs the caller's partials
    lib.hb_softmax_xent.argtypes = [P, i64, i32, i32, P, P, ctypes.c_double, P, i64, P, P, i32, P, P]
    rc = lib.hb_softmax_xent(16, 8, 20000, 8, 16, 16, 1.0, 16, 8, 16, 16, 0, None, None)
    assert rc == -1 and b"hb_softmax_xent" in lib.hb_last_error()
