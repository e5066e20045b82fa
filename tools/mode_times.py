"""GPU time of each single mode product of a Tucker shape (CUDA-graph replay,
no host overhead) and the HBM bytes it moves: which modes of a small-extent
high-order tensor fall short of the memory roofline. argv: shape, e.g. 20x20x20x20x20x20."""
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
for arg in sys.argv[1].split(","):
    shape = tuple(int(x) for x in arg.split("x"))
    d = len(shape)
    T = mm.colmajor_empty(shape, torch.float64, "cuda").normal_()
    S = torch.empty_like(T)
    L = mm.to_colmajor(torch.randn(shape[0], shape[0], dtype=torch.float64, device="cuda"))
    m = _lib.i64_array(shape)
    row = []
    for mu in range(1, d + 1):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            h.bind_torch_stream()
            for _ in range(2):
                assert lib.mumode_mode_product_f64(h.h, d, m, mu, shape[mu - 1], T.data_ptr(), L.data_ptr(),
                                                   S.data_ptr()) == 0
            with torch.cuda.graph(g, stream=s):
                for _ in range(10):
                    lib.mumode_mode_product_f64(h.h, d, m, mu, shape[mu - 1], T.data_ptr(), L.data_ptr(),
                                                S.data_ptr())
        torch.cuda.synchronize()
        h.bind_torch_stream()
        g.replay()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / 10 * 1e3
        row.append(f"mode {mu}: {us:.1f} us {2 * T.numel() * 8 / us / 1e6:.2f} TB/s")
    print(arg, " | ".join(row), flush=True)
