"""Tucker chains per-mode (policy 0) vs one persistent chain launch (policy
11): launches per application, bitwise equality, time."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402
from odd_modes import timeit  # noqa: E402

h = mm.get_handle(0)
cases = [((256, 256, 256), (256, 256, 256), False), ((200, 200, 200), (200, 200, 200), False),
         ((128, 128, 128), (192, 192, 192), True), ((96, 512, 384), (128, 128, 128), False),
         ((64, 64, 64, 64), (64, 64, 64, 64), False), ((512, 512, 64), (512, 512, 64), False)]
for m, n, cplx in cases:
    dt = torch.complex128 if cplx else torch.float64
    T = mm.colmajor_empty(m, dt, "cuda")
    T.copy_(torch.randn(m, dtype=dt, device="cuda"))
    Ls = [mm.to_colmajor(torch.randn(n[k], m[k], dtype=dt, device="cuda")) for k in range(len(m))]
    fl = sum(2 * n[k] * (8 if cplx else 1) / (4 if cplx else 1) for k in range(len(m)))  # placeholder
    row = {"m": m, "n": n, "cplx": cplx}
    out = {}
    for pol in (0, 11):
        h.set_kernel_policy(pol)
        S = mm.tucker(T, Ls)
        torch.cuda.synchronize()
        l0 = h.launches
        S = mm.tucker(T, Ls)
        torch.cuda.synchronize()
        row[f"launches_p{pol}"] = h.launches - l0
        out[pol] = S.clone()
        row[f"ms_p{pol}"] = round(timeit(lambda: mm.tucker(T, Ls)), 4)
    h.set_kernel_policy(0)
    row["bitwise"] = bool(torch.equal(out[0], out[11]))
    row["gain_pct"] = round(100 * (row["ms_p0"] / row["ms_p11"] - 1), 2)
    print(json.dumps(row))
