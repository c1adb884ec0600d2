"""cuBLAS DGEMM ceiling (torch.matmul float64) — cross-check for the FP64 roofline denominator."""
import json, torch
torch.backends.cuda.matmul.allow_tf32 = False
for n in (1024, 4096, 8192):
    a = torch.rand(n, n, dtype=torch.float64, device="cuda")
    b = torch.rand(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20 if n < 8192 else 5
    e0.record()
    for _ in range(reps):
        c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"bench": "cublas_dgemm", "n": n, "ms": ms, "tflops": 2 * n**3 / ms / 1e9}))
