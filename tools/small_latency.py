"""Latency of small Tucker calls (config C1, 100 x 100): host wall time per
Python API call, per C-ABI call (ctypes, preallocated), and the GPU time of
the same launches replayed from a CUDA graph."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402
from paper_2112_11238_b200 import _lib  # noqa: E402

lib = _lib.lib()
h = mm.get_handle(0)
h.bind_torch_stream()
T = mm.colmajor_empty((100, 100), torch.float64, "cuda").normal_()
Ls = [mm.to_colmajor(torch.randn(100, 100, dtype=torch.float64, device="cuda")) for _ in range(2)]
S = mm.colmajor_empty((100, 100), torch.float64, "cuda")
m = _lib.i64_array((100, 100))
P = _lib.ptr_array([L.data_ptr() for L in Ls])
N = 2000


def wall(fn):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / N * 1e6


print(f"python mm.tucker   : {wall(lambda: mm.tucker(T, Ls)):.2f} us per call")
print(f"C-ABI tucker_f64   : {wall(lambda: lib.mumode_tucker_f64(h.h, 2, m, m, T.data_ptr(), P, S.data_ptr(), 0)):.2f} us per call")
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    h.bind_torch_stream()
    lib.mumode_tucker_f64(h.h, 2, m, m, T.data_ptr(), P, S.data_ptr(), 0)
    with torch.cuda.graph(g, stream=s):
        for _ in range(100):
            lib.mumode_tucker_f64(h.h, 2, m, m, T.data_ptr(), P, S.data_ptr(), 0)
torch.cuda.synchronize()
h.bind_torch_stream()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
g.replay()
a.record()
for _ in range(10):
    g.replay()
b.record()
torch.cuda.synchronize()
print(f"graph replay       : {a.elapsed_time(b) / 1000 * 1e3:.2f} us per Tucker (GPU time, 2 launches)")
