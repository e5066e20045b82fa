"""Repeat each complex mode product of C4 (and each forced complex tile
config) and count runs that differ from the first: localises a
non-deterministic complex kernel."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402

torch.manual_seed(0)
h = mm.get_handle(0)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
T1 = mm.colmajor_empty((128, 128, 128), torch.complex128, "cuda").normal_()
T2 = mm.colmajor_empty((192, 128, 128), torch.complex128, "cuda").normal_()
T3 = mm.colmajor_empty((192, 192, 128), torch.complex128, "cuda").normal_()
L = mm.to_colmajor(torch.randn(192, 128, dtype=torch.complex128, device="cuda"))
for pol in (0, 3, 4, 5, 6):
    h.set_kernel_policy(pol)
    out = []
    for mu, T in ((1, T1), (2, T2), (3, T3)):
        first = mm.mode_product(T, L, mu).clone()
        nbad = 0
        rows = set()
        for _ in range(reps):
            S = mm.mode_product(T, L, mu)
            if not torch.equal(S, first):
                nbad += 1
                d = (S != first).nonzero()
                rows.update(int(x) for x in d[:, 0].unique()[:4])
        out.append(f"mode {mu}: {nbad}/{reps} differ" + (f" rows {sorted(rows)[:8]}" if rows else ""))
    print(f"policy {pol}: " + " | ".join(out), flush=True)
h.set_kernel_policy(0)
