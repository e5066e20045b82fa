"""C3: 100 exponential-integrator steps on 200^3 (one CUDA graph), ms per
100 steps (median of 5, L2 flushed) and a checksum for bitwise comparison
between builds / tile policies."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402

torch.manual_seed(0)
A = torch.zeros(200, 200, dtype=torch.float64)
hh = 1.0 / 201
for i in range(200):
    A[i, i] = -2 / hh ** 2
    if i > 0:
        A[i, i - 1] = 1 / hh ** 2 - 0.5 / (2 * hh)
    if i < 199:
        A[i, i + 1] = 1 / hh ** 2 + 0.5 / (2 * hh)
E = torch.from_numpy(mm.expm((1e-3 * A).numpy())).cuda()
u0 = mm.colmajor_empty((200, 200, 200), torch.float64, "cuda").normal_()
u1 = mm.colmajor_empty((200, 200, 200), torch.float64, "cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
mm.expint(u0, [E, E, E], 100, out=u1)
ts = []
for _ in range(5):
    flush.fill_(1.0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    mm.expint(u0, [E, E, E], 100, out=u1)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = sorted(ts)[2]
flops = 100 * 3 * 2 * 200 ** 4
x = u1.cpu().numpy()
print(f"C3 100 steps: {ms:.3f} ms  {flops / ms / 1e9:.1f} GF/s  checksum {np.float64(x.sum()).hex()} {np.float64((x * x).sum()).hex()}")
