"""Short run for ncu: C2 Tucker (256^3) then C3-shaped Tucker (200^3), two
warm-up applications each, then one profiled (3 mode-product launches each)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402

for n in (256, 200):
    T = mm.colmajor_empty((n, n, n), torch.float64, "cuda").normal_()
    Ls = [mm.to_colmajor(torch.randn(n, n, dtype=torch.float64, device="cuda")) for _ in range(3)]
    for _ in range(3):
        S = mm.tucker(T, Ls)
    torch.cuda.synchronize()
    print("ok", n, float(S.abs().max()))
