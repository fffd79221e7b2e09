"""Debug harness for the TMA GEMM (not a test)."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from paper_2303_01277_b200 import ops, _lib
lib = _lib.load()
lib.hb_gemm_debug_buffer.argtypes = [ctypes.c_void_p, ctypes.c_int]
for mode, (M, N, K, kind) in [(-1, (128, 64, 32, "kk")), (0, (128, 64, 32, "kk")), (2, (128, 64, 32, "kk")), (0, (128, 64, 32, "nn")),
                              (0, (128, 256, 32, "nn"))]:
    BN = 64 if N <= 64 else 256
    stage = 2 * (128 * 32 * 4 + BN * 32 * 4) // 4
    dbg = torch.zeros(stage + 16, dtype=torch.int32, device="cuda")
    lib.hb_gemm_debug_buffer(dbg.data_ptr() if mode >= 0 else None, max(mode, 0))
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(M, K, device="cuda", generator=g)
    B = torch.randn(N, K, device="cuda", generator=g).t() if kind == "kk" else torch.randn(K, N, device="cuda", generator=g)
    C = torch.full((M, N), 7.0, device="cuda")
    ops.gemm(A, B, C)
    torch.cuda.synchronize()
    d = dbg.cpu().numpy().view(np.uint32)
    ref = A @ B
    print(f"mode {mode} {kind} M{M} N{N} K{K}: err {(C - ref).abs().max().item():.3e}  C00 {C[0,0].item():.4f} ref {ref[0,0].item():.4f}")
    print("   marker %x tmem %x idesc %x pad %x descA %08x_%08x descB %08x_%08x st %x" % tuple(int(x) for x in d[stage:stage + 9]))
lib.hb_gemm_debug_buffer(None, 0)
