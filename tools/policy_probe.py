"""Run a Tucker of one shape under one kernel policy (diagnostics)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402

h = mm.get_handle(0)
shape = tuple(int(x) for x in sys.argv[1].split("x"))
h.set_kernel_policy(int(sys.argv[2]))
torch.manual_seed(1)
T = mm.colmajor_empty(shape, torch.float64, "cuda").normal_()
Ls = [mm.to_colmajor(torch.randn(e, e, dtype=torch.float64, device="cuda")) for e in shape]
S = mm.tucker(T, Ls)
torch.cuda.synchronize()
print(shape, "policy", sys.argv[2], "ok", float(S.abs().max()), flush=True)
