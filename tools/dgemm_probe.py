"""cuBLAS DGEMM yardstick (torch float64 matmul) on the box: 8192^3 and the
C2-shaped products. Library numbers are a yardstick only, never the product."""
import json
import torch


def bench(f, flops, reps=10):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        e0.record()
        f()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best, flops / best / 1e9


dev = "cuda"
a = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
b = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
ms, tf = bench(lambda: a @ b, 2 * 8192**3)
print(json.dumps({"variant": "cublas_dgemm_8192", "ms": ms, "tflops": tf}))
L = torch.randn(256, 256, dtype=torch.float64, device=dev)
T = torch.randn(256, 65536, dtype=torch.float64, device=dev)
ms, tf = bench(lambda: L @ T, 2 * 256 * 256 * 65536)
print(json.dumps({"variant": "cublas_mode1_256", "ms": ms, "tflops": tf}))
Tb = torch.randn(256, 256, 256, dtype=torch.float64, device=dev)
ms, tf = bench(lambda: torch.matmul(Tb, L.t()), 2 * 256 * 256 * 65536)
print(json.dumps({"variant": "cublas_batched_256", "ms": ms, "tflops": tf}))
# sustained: 3 s of back-to-back 8192^3
import time
torch.cuda.synchronize()
t0 = time.time()
n = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 3.0:
    for _ in range(5):
        a @ b
        n += 1
    torch.cuda.synchronize()
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1)
print(json.dumps({"variant": "cublas_dgemm_8192_sustained", "n": n, "tflops": 2 * 8192**3 * n / ms / 1e9}))
