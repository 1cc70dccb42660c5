"""FP64 roofline denominator: cuBLAS DGEMM 8192^3 (torch.matmul, best of 10) plus the
DFMA / DMMA microbenchmarks of scripts/fp64_peak.cu (build/fp64_peak, built here with
nvcc).  Prints one JSON line; profiles/fp64_peak_r01.json keeps the measured copy."""
import json
import os
import subprocess

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
c = a @ b
best = 1e30
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    c = a @ b
    e.record()
    torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
out = {"dgemm_8192_tflops": 2.0 * n ** 3 / best / 1e9, "dgemm_ms": best}
exe = os.path.join(ROOT, "build", "fp64_peak")
if os.path.exists(exe):
    for line in subprocess.run([exe], capture_output=True, text=True).stdout.splitlines():
        if line.startswith("{"):
            d = json.loads(line)
            out[d["probe"] + "_tflops"] = d["tflops"]
out["fp64_peak_tflops"] = max(v for k, v in out.items() if k.endswith("_tflops"))
out["gpu"] = torch.cuda.get_device_name(0)
print(json.dumps(out))
