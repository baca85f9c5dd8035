"""Measure the FP64 roofline denominators on the B200 box -> profiles/fp64_peak.json.

DFMA pipe and DMMA (mma.sync m8n8k4 f64) microbenchmarks (tools/fp64_peak.cu), plus cuBLAS
DGEMM through torch.matmul at 8192^3 (same method as MEASURED_PEAKS.json's bf16 entry)."""
import ctypes
import json
import os
import subprocess
import time

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
so = os.path.join(HERE, "libfp64peak.so")
if not os.path.exists(so):
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-Xcompiler", "-fPIC", "-shared", "-o", so, os.path.join(HERE, "fp64_peak.cu")])
lib = ctypes.CDLL(so)
a, b = ctypes.c_double(), ctypes.c_double()
best_f = best_m = 0.0
for _ in range(5):
    assert lib.fp64_peak(ctypes.byref(a), ctypes.byref(b)) == 0
    best_f, best_m = max(best_f, a.value), max(best_m, b.value)
N = 8192
A = torch.randn(N, N, dtype=torch.float64, device="cuda")
B = torch.randn(N, N, dtype=torch.float64, device="cuda")
for _ in range(2):
    A @ B
torch.cuda.synchronize()
best = 0.0
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    A @ B
    e1.record()
    torch.cuda.synchronize()
    best = max(best, 2 * N ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
out = {"fp64_fma_tflops": best_f, "fp64_dmma_tflops": best_m, "fp64_dgemm_cublas_tflops": best,
       "gpu": torch.cuda.get_device_name(), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
       "how": "tools/fp64_peak.py: DFMA chains (8 indep/thread, 148*8 CTAs x 256 thr), mma.sync m8n8k4 f64 "
              "(8 indep accumulators/warp), torch.matmul fp64 8192^3 best of 5"}
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "profiles", "fp64_peak.json"), "w"), indent=1)
print(json.dumps(out))
