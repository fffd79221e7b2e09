"""ctypes binding of the C-ABI library ``libhalob200.so`` (include/halob200.h).

There is no fallback: if the library is missing or no CUDA device is present,
every device entry point raises.  The library is built in-tree by
``__graft_entry__.build()`` (``make -C paper_2303_01277_b200/csrc``).
"""

from __future__ import annotations

import ctypes
from ctypes import c_double, c_float, c_int32, c_int64, c_uint32, c_uint64, c_void_p
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libhalob200.so"

HB_OK, HB_EINVAL, HB_ECUDA = 0, -1, -2
HB_FLAG_NONFINITE = 1
HEADER_BYTES = 12

# hb_segment_t (40 bytes): key0, key1, elem_offset, out, row_begin, num_rows
SEGMENT_DTYPE = np.dtype([("key0", "<u8"), ("key1", "<u8"), ("elem_offset", "<u8"),
                          ("out", "<u8"), ("row_begin", "<i4"), ("num_rows", "<i4")])
assert SEGMENT_DTYPE.itemsize == 40

EXPORTS = (
    "hb_version", "hb_last_error", "hb_philox_uniforms", "hb_quantize_gather",
    "hb_dequant_gather", "hb_spmm_csr", "hb_spmm_csr_ex", "hb_spmm_tiled", "hb_spmm_tiled_bin", "hb_gemm_f32", "hb_gemm2_f32", "hb_gemm_set_path", "hb_spmm_set_narrow", "hb_softmax_xent", "hb_relu", "hb_relu_grad_mul",
    "hb_adam_step", "hb_adam_step_guarded", "hb_adam_step_dev", "hb_upload_async", "hb_ipc_get_handle", "hb_ipc_open_handle",
    "hb_ipc_close", "hb_p2p_signal", "hb_p2p_wait", "hb_argmax_accuracy", "hb_dropout", "hb_sigmoid_bce", "hb_multilabel_counts",
)

P = c_void_p
_SIGS = {
    "hb_philox_uniforms": [c_uint64, c_uint64, c_uint64, c_int64, P, P],
    "hb_quantize_gather": [P, c_int64, P, c_int32, P, c_int32, c_int32, c_int32, P, P],
    "hb_dequant_gather": [P, c_int32, c_int32, P, P, P, c_int32, c_int32, P, c_int64, c_int32, P],
    "hb_spmm_csr": [c_int32, P, P, P, P, c_int64, c_int32, P, c_int64, P],
    "hb_gemm_f32": [c_int32, c_int32, c_int32, P, c_int64, c_int64, P, c_int64, c_int64, P, c_int64,
                    c_float, P, c_int64, P, c_int64, P],
    "hb_gemm2_f32": [c_int32, c_int32, c_int32, P, c_int64, c_int64, P, c_int64, c_int64, c_int32, P, c_int64,
                     c_int64, P, c_int64, c_int64, P, c_int64, c_float, P, c_int64, P, c_int64, P],
    "hb_gemm_set_path": [c_int32],
    "hb_spmm_set_narrow": [c_int32],
    "hb_spmm_tiled": [c_int32, c_int32, c_int32, P, P, P, P, P, P, P, P, P, c_int64, c_int32, P, c_int64, P, P],
    "hb_spmm_tiled_bin": [c_int32, c_int32, c_int32, P, P, P, P, P, P, P, P, P, P, c_int64, c_int32, P, c_int64,
                          P, c_int64, P, c_int32, c_int32, P, P],
    "hb_spmm_csr_ex": [c_int32, P, P, P, P, c_int64, c_int32, P, c_int64, c_int64, c_int32, c_int32, c_int32, P, P],
    "hb_softmax_xent": [P, c_int64, c_int32, c_int32, P, P, c_double, P, c_int64, P, P, c_int32, P, P],
    "hb_relu": [P, c_int64, c_int32, c_int32, P, c_int64, P],
    "hb_sigmoid_bce": [P, c_int64, c_int32, c_int32, P, c_int64, P, c_double, P, c_int64, P, P, c_int32, P, P],
    "hb_multilabel_counts": [P, c_int64, c_int32, c_int32, P, c_int64, P, P, P],
    "hb_relu_grad_mul": [P, c_int64, P, c_int64, c_int32, c_int32, P, c_int64, P],
    "hb_adam_step": [P, P, P, P, c_int64, c_float, c_float, c_float, c_float, c_double, c_double, P],
    "hb_adam_step_guarded": [P, P, P, P, c_int64, c_float, c_float, c_float, c_float, c_double, c_double, P, P, P,
                             P],
    "hb_upload_async": [P, P, c_int64, P],
    "hb_ipc_get_handle": [P, P, P],
    "hb_ipc_open_handle": [P, P],
    "hb_ipc_close": [P],
    "hb_p2p_signal": [P, c_int32, P],
    "hb_p2p_wait": [P, c_uint64, P, P, c_uint32, c_uint64, P],
    "hb_adam_step_dev": [P, P, P, P, c_int64, c_float, c_float, c_float, c_float, P, P, P, P, P],
    "hb_argmax_accuracy": [P, c_int64, c_int32, c_int32, P, P, P, P],
    "hb_dropout": [P, c_int64, c_int32, c_int64, c_int32, c_uint64, c_uint64, c_float, P, c_int64, P],
}


class HaloLibError(RuntimeError):
    """A C-ABI call failed (HB_ECUDA or an unexpected code)."""


class HaloArgError(ValueError):
    """A C-ABI call rejected its arguments (HB_EINVAL)."""


_lib = None


def load(path: Path | None = None) -> ctypes.CDLL:
    """Load (once) and type the library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise HaloLibError(f"{p} is missing: build it with __graft_entry__.build() "
                           "(there is no CPU fallback for the halo path)")
    lib = ctypes.CDLL(str(p))
    lib.hb_version.restype = ctypes.c_char_p
    lib.hb_last_error.restype = ctypes.c_char_p
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = c_int32
    _lib = lib
    return lib


def call(name: str, *args):
    rc = getattr(load(), name)(*args)
    if rc != HB_OK:
        msg = load().hb_last_error().decode(errors="replace")
        if rc == HB_EINVAL:
            raise HaloArgError(f"{name}: {msg}")
        raise HaloLibError(f"{name} failed ({rc}): {msg}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
