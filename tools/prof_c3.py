"""C3-shaped Tucker (200^3, E from the reference's stencil) for ncu: 3 warm-up
applications + 1 profiled one."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402

g = mm.Rng(1234)
u = torch.from_numpy(g.normal((200, 200, 200))).cuda()
E = torch.from_numpy(np.asfortranarray(g.normal((200, 200)) * 0.07)).cuda()
for _ in range(4):
    S = mm.tucker(u, [E, E, E])
torch.cuda.synchronize()
print("ok", float(S.abs().max()))
