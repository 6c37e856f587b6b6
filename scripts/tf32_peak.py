#!/usr/bin/env python
"""Measure the B200's dense TF32 tensor-core peak (the roofline denominator of
the 3xTF32 GEMMs, SURVEY.md §7 hard part 1): fp32 torch.matmul with TF32
tensor cores (cuBLAS), 8192^3, best of 10 (burst) and back to back for 4 s
(sustained), same recipe as MEASURED_PEAKS.json's bf16 figure.  Also the
plain FP32 (no TF32) SIMT rate for reference.

    python scripts/tf32_peak.py profiles/r02_tf32_peak.json
"""

import json
import subprocess
import sys
import time

import torch


def rate(n, dtype, tf32, reps=10, sustain_s=0.0):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    torch.backends.cudnn.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    c = torch.empty(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = max(best, 2.0 * n ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
    sustained = None
    if sustain_s > 0:
        t_end = time.perf_counter() + sustain_s
        k = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        while time.perf_counter() < t_end:
            for _ in range(20):
                torch.matmul(a, b, out=c)
            k += 20
            torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        sustained = 2.0 * n ** 3 * k / (e0.elapsed_time(e1) / 1e3) / 1e12
    return best, sustained


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "profiles/r02_tf32_peak.json"
    clocks = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,name", "--format=csv,noheader"],
                            capture_output=True, text=True).stdout.strip()
    tb, ts = rate(8192, torch.float32, True, sustain_s=4.0)
    fb, _ = rate(8192, torch.float32, False, reps=3)
    bb, _ = rate(8192, torch.bfloat16, False)
    d = {"tf32_tflops_burst": round(tb, 1), "tf32_tflops_sustained": round(ts, 1),
         "fp32_simt_tflops_burst": round(fb, 1), "bf16_tflops_burst_same_run": round(bb, 1),
         "how": "torch.matmul 8192^3 fp32 with allow_tf32 (cuBLAS TF32 tensor cores): best of 10 (burst) and back to "
                "back for 4 s (sustained); fp32 SIMT = allow_tf32 off; bf16 for comparison with MEASURED_PEAKS.json",
         "nvidia_smi_after": clocks, "torch": torch.__version__, "device": torch.cuda.get_device_name(0)}
    with open(out, "w") as f:
        json.dump(d, f, indent=1)
    print(json.dumps(d))


if __name__ == "__main__":
    main()
