"""DMMA GEMM microbenchmark (diagnostic): library gemm_batched (spd_test_gemm, one
descriptor) vs torch.matmul fp64 (cuBLAS DGEMM) on square and QR/H2-like shapes.
usage: SPD_GEMM_TILE=64|128 python tools/gemm_bench.py"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_07632_b200 as spd  # noqa: E402

lib = spd.lib()
shapes = [(0, 0, 4096, 4096, 4096), (1, 0, 4096, 4096, 4096), (0, 1, 4096, 4096, 4096), (1, 1, 4096, 4096, 4096),
          (0, 0, 8192, 8192, 1024), (0, 0, 6144, 1024, 32), (1, 0, 32, 1024, 6144), (0, 0, 32768, 110, 2048),
          (1, 0, 2048, 110, 32768)]


def t_of(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for ta, tb, m, n, k in shapes:
    A = torch.randn((k, m) if ta else (m, k), dtype=torch.float64, device="cuda")
    B = torch.randn((n, k) if tb else (k, n), dtype=torch.float64, device="cuda")
    C = torch.zeros((n, m), dtype=torch.float64, device="cuda")      # col-major m x n
    Ac = A.t().contiguous() if True else A    # storage col-major: (rows, cols) -> transpose contiguous
    Bc = B.t().contiguous()
    lda, ldb = A.shape[0], B.shape[0]

    def ours():
        st = lib.spd_test_gemm(ta, tb, m, n, k, 1.0, ctypes.c_void_p(Ac.data_ptr()), lda,
                               ctypes.c_void_p(Bc.data_ptr()), ldb, 0.0, ctypes.c_void_p(C.data_ptr()), m,
                               spd._stream())
        assert st == 0, lib.spd_last_error()

    def ref():
        return (A.t() if ta else A) @ (B.t() if tb else B)

    to, tr = t_of(ours), t_of(ref)
    fl = 2.0 * m * n * k
    err = (C.t() - ref()).abs().max().item() / max(1e-300, ref().abs().max().item())
    print(f"ta={ta} tb={tb} {m}x{n}x{k}: ours {to:8.3f} ms {fl/to/1e9:7.2f} TF | cuBLAS {tr:8.3f} ms "
          f"{fl/tr/1e9:7.2f} TF | rel err {err:.1e}", flush=True)
