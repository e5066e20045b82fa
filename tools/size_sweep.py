"""Tucker TF/s on even cubes (all TMA-legal) and per-config forced policies:
where does the tile cost model leave throughput behind?"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402
from timing import timeit  # noqa: E402

h = mm.get_handle(0)
sizes = [int(a) for a in sys.argv[1:]] or [96, 128, 160, 192, 200, 224, 240, 256, 272, 288, 320, 352, 384, 448, 512]
for n in sizes:
    T = mm.colmajor_empty((n, n, n), torch.float64, "cuda").normal_()
    Ls = [mm.to_colmajor(torch.randn(n, n, dtype=torch.float64, device="cuda")) for _ in range(3)]
    row = {"n": n}
    for pol in (0, 3, 4, 5, 6):
        h.set_kernel_policy(pol)
        ms = timeit(lambda: mm.tucker(T, Ls))
        row[f"p{pol}"] = round(3 * 2 * n ** 4 / ms / 1e9, 1)
    h.set_kernel_policy(0)
    print(json.dumps(row))
