"""Auto-policy Tucker throughput over n^3 cubes (fp64, device-resident, median
of 10): TF/s and % of the 37.0 TF/s fp64 roofline, to find the extents the
tile configurations serve worst. python tools/auto_sweep.py [lo hi step]"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import paper_2112_11238_b200 as mm  # noqa: E402
from timing import timeit  # noqa: E402

lo, hi, step = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (96, 512, 8)
for n in range(lo, hi + 1, step):
    T = mm.colmajor_empty((n, n, n), torch.float64, "cuda").normal_()
    Ls = [mm.to_colmajor(torch.randn(n, n, dtype=torch.float64, device="cuda")) for _ in range(3)]
    ms = timeit(lambda: mm.tucker(T, Ls))
    tf = 3 * 2 * n ** 4 / ms / 1e9
    print(json.dumps({"n": n, "tf": round(tf, 1), "pct": round(100 * tf / 37.0, 1)}), flush=True)
    del T
