"""Measure the B200 FP64 roofline denominators that MEASURED_PEAKS.json lacks:
cuBLAS DGEMM (torch.matmul float64) 8192^3 best of 10 (burst) and back to back
for 4 s (sustained), with SM clocks sampled.  Writes profiles/fp64_peak.json."""
import json
import os
import subprocess
import time

import torch


def main():
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); torch.matmul(a, b); e.record(); e.synchronize()
        best = max(best, 2 * n ** 3 / (s.elapsed_time(e) * 1e-3) / 1e12)
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks_event_reasons.active", "--format=csv,noheader,nounits",
                            "-lms", "200", "-i", str(torch.cuda.current_device())], stdout=subprocess.PIPE, text=True)
    t0 = time.time(); cnt = 0
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    while time.time() - t0 < 4.0:
        torch.matmul(a, b); cnt += 1
        if cnt % 8 == 0:
            torch.cuda.synchronize()
    e.record(); e.synchronize()
    smi.terminate()
    out = smi.communicate()[0].strip().splitlines()
    clocks = [int(l.split(",")[0]) for l in out if l.split(",")[0].strip().isdigit()]
    sus = 2 * n ** 3 * cnt / (s.elapsed_time(e) * 1e-3) / 1e12
    res = {"fp64_dgemm_tflops": round(best, 2), "fp64_dgemm_tflops_sustained": round(sus, 2),
           "how": "torch.matmul float64 (cuBLAS DGEMM) 8192^3: best of 10 and back-to-back 4 s",
           "sm_mhz_median_sustained": sorted(clocks)[len(clocks) // 2] if clocks else None,
           "gpu": torch.cuda.get_device_name(), "torch": torch.__version__,
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    os.makedirs("profiles", exist_ok=True)
    json.dump(res, open("profiles/fp64_peak.json", "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
