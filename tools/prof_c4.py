"""Short C4 (complex 128^3 -> 192^3) run for ncu."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402

T = mm.colmajor_empty((128,) * 3, torch.complex128, "cuda").normal_()
Ls = [mm.to_colmajor(torch.randn(192, 128, dtype=torch.complex128, device="cuda")) for _ in range(3)]
for _ in range(3):
    S = mm.tucker(T, Ls)
torch.cuda.synchronize()
print("ok", float(S.abs().max()))
