"""IMEX direct solve (DirectSolver::solve, src/imex.cpp:67-86) at 200^3:
two Tuckers around the eigen-sum division, device-resident."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle as O  # noqa: E402  (problem setup only: the stencil)
import paper_2112_11238_b200 as mm  # noqa: E402
from odd_modes import timeit  # noqa: E402

n = 200
M = np.eye(n) / 3 - 1e-3 * O.port_advection_diffusion(n, 0.0)
solver = mm.KronSumSolver(Ms=[M, M, M])
b = torch.from_numpy(mm.Rng(1).normal((n, n, n))).cuda()
for pol in (0, 8):
    mm.get_handle(0).set_kernel_policy(pol)
    ms = timeit(lambda: solver.solve(b))
    print(f"policy {pol}: solve {ms:.4f} ms  ({2 * 3 * 2 * n ** 4 / ms / 1e9:.1f} TFLOP/s of Tucker work)")
mm.get_handle(0).set_kernel_policy(0)
