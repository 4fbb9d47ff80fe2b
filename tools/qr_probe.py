"""Blocked-QR probe (diagnostic): time spd_test_qr_unpivoted on H2-build-like batches
and print the library's per-kernel-class profile.  usage: python tools/qr_probe.py [B m n] ..."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_07632_b200 as spd  # noqa: E402
from bench import prof_table  # noqa: E402

cases = [(256, 6144, 128), (128, 6144, 256), (32, 6144, 988), (16, 6144, 1480)]
if len(sys.argv) > 3:
    a = list(map(int, sys.argv[1:]))
    cases = [tuple(a[i:i + 3]) for i in range(0, len(a), 3)]
lib = spd.lib()
for B, m, n in cases:
    A = torch.randn(B, n, m, dtype=torch.float64, device="cuda")
    for rep in range(3):
        X = A.clone()
        torch.cuda.synchronize()
        if rep == 2:
            lib.spd_prof_reset()
            lib.spd_prof_enable(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = lib.spd_test_qr_unpivoted(B, ctypes.c_void_p(X.data_ptr()), m, n, m, m * n, spd._stream())
        e1.record()
        torch.cuda.synchronize()
        assert st == 0, lib.spd_last_error()
        if rep >= 1:
            fl = B * (2.0 * m * n * n - 2.0 / 3.0 * n ** 3)
            ms = e0.elapsed_time(e1)
            print(f"B={B} m={m} n={n}: {ms:.2f} ms  {fl / ms / 1e9:.2f} TF/s", flush=True)
    lib.spd_prof_enable(0)
    for k, v in sorted(prof_table(lib).items(), key=lambda kv: -kv[1]["ms"]):
        print(f"   {k:14s} {int(v['launches']):5d} {v['ms']:9.2f} ms")
