"""Odd cubes: padded TMA chain (policy 0) vs LDG-staged DMMA (policy 8)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402
from timing import timeit  # noqa: E402

h = mm.get_handle(0)
for n in [int(a) for a in sys.argv[1:]] or (97, 129, 143, 161, 175, 191, 201, 223, 239, 255, 289, 321, 383):
    T = mm.colmajor_empty((n, n, n), torch.float64, "cuda").normal_()
    Ls = [mm.to_colmajor(torch.randn(n, n, dtype=torch.float64, device="cuda")) for _ in range(3)]
    row = {"n": n}
    for pol in (0, 8):
        h.set_kernel_policy(pol)
        ms = timeit(lambda: mm.tucker(T, Ls))
        row[f"p{pol}_tf"] = round(3 * 2 * n ** 4 / ms / 1e9, 1)
    h.set_kernel_policy(0)
    print(json.dumps(row))
