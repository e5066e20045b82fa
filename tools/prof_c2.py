"""Short C2 run for ncu: 2 warm-up Tucker applications + 1 profiled one
(3 TMA/DMMA mode-product launches per application)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402

g = mm.Rng(1234)
T = torch.from_numpy(g.normal((256, 256, 256))).cuda()
Ls = [torch.from_numpy(g.normal((256, 256))).cuda() for _ in range(3)]
for _ in range(3):
    S = mm.tucker(T, Ls)
torch.cuda.synchronize()
print("ok", float(S.abs().max()))
