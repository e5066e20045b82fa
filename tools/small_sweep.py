"""GPU time of small Tucker operators (CUDA-graph replay of 20 C-ABI calls,
so host overhead is excluded): the tile choice for products of a few tiles.
Shapes: argv (e.g. 100x100,32x32x32) or a default list."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402
from paper_2112_11238_b200 import _lib  # noqa: E402

lib = _lib.lib()
h = mm.get_handle(0)
import os  # noqa: E402
h.set_kernel_policy(int(os.environ.get("POLICY", "0")))
shapes = [tuple(int(x) for x in s.split("x")) for s in sys.argv[1].split(",")] if len(sys.argv) > 1 else \
    [(100, 100), (256, 256), (512, 512), (16,) * 3, (32,) * 3, (48,) * 3, (64,) * 3, (80,) * 3, (96,) * 3,
     (128,) * 3, (160,) * 3]
out = []
for shape in shapes:
    d = len(shape)
    T = mm.colmajor_empty(shape, torch.float64, "cuda").normal_()
    Ls = [mm.to_colmajor(torch.randn(e, e, dtype=torch.float64, device="cuda")) for e in shape]
    S = mm.colmajor_empty(shape, torch.float64, "cuda")
    m = _lib.i64_array(shape)
    P = _lib.ptr_array([L.data_ptr() for L in Ls])
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        h.bind_torch_stream()
        for _ in range(3):
            assert lib.mumode_tucker_f64(h.h, d, m, m, T.data_ptr(), P, S.data_ptr(), 0) == 0
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                lib.mumode_tucker_f64(h.h, d, m, m, T.data_ptr(), P, S.data_ptr(), 0)
    torch.cuda.synchronize()
    h.bind_torch_stream()
    g.replay()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 20 * 1e3)
    flops = sum(2 * shape[k] * int(torch.tensor(shape).prod()) for k in range(d))
    out.append(f"{'x'.join(map(str, shape))}: {best:.2f} us ({flops / best / 1e6:.2f} TF/s)")
print("  ".join(out))
