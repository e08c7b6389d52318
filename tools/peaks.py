"""Measured dense peaks for the roofline denominators that MEASURED_PEAKS.json does not carry (VERDICT r1
item 6), with its protocol: cuBLAS (torch.matmul) 8192^3, best of 10 (burst) and back to back for 4 s
(sustained), CUDA events.  TF32 (allow_tf32) and FP32 SIMT (allow_tf32 off).  Plus the HBM copy figure
for a same-box cross-check.  Writes one JSON object to stdout.

    python tools/peaks.py > profiles/peaks_r2.json
"""
import json
import time

import torch


def mm_peaks(allow_tf32, n=8192, sustain_s=4.0):
    torch.backends.cuda.matmul.allow_tf32 = allow_tf32
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    c = torch.empty(n, n, device="cuda")
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(10):
        e0.record(); torch.matmul(a, b, out=c); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    flops = 2.0 * n ** 3
    burst = flops / (best / 1e3) / 1e12
    reps, t0 = 0, time.time()
    e0.record()
    while time.time() - t0 < sustain_s:
        for _ in range(10):
            torch.matmul(a, b, out=c)
        reps += 10
        torch.cuda.synchronize()
    e1.record(); e1.synchronize()
    sustained = flops * reps / (e0.elapsed_time(e1) / 1e3) / 1e12
    return burst, sustained


def hbm_copy():
    a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
    b = torch.empty_like(a)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(10):
        e0.record(); b.copy_(a); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return 2.0 * a.numel() * 2 / (best / 1e3) / 1e9


if __name__ == "__main__":
    tf_b, tf_s = mm_peaks(True)
    fp_b, fp_s = mm_peaks(False, sustain_s=2.0)
    out = {"tf32_tflops": tf_b, "tf32_tflops_sustained": tf_s, "fp32_simt_tflops": fp_b,
           "fp32_simt_tflops_sustained": fp_s, "hbm_copy_gbs": hbm_copy(),
           "gpu_name": torch.cuda.get_device_name(0), "torch": torch.__version__,
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "how": "torch.matmul fp32 8192^3 (2 N^3) with allow_tf32 on (TF32) / off (FP32 SIMT): best of 10 "
                  "(burst) and back to back for 4 s / 2 s (sustained); HBM: bf16 copy of 1 Gi elements, best "
                  "of 10 (read + write bytes)"}
    print(json.dumps(out, indent=1))
