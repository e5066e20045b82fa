"""Short 20^6 Tucker run for ncu (six skinny mode products)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402

T = mm.colmajor_empty((20,) * 6, torch.float64, "cuda").normal_()
Ls = [mm.to_colmajor(torch.randn(20, 20, dtype=torch.float64, device="cuda")) for _ in range(6)]
for _ in range(3):
    S = mm.tucker(T, Ls)
torch.cuda.synchronize()
print("ok", float(S.abs().max()))
