"""Auto-policy complex128 Tucker throughput over n^3 cubes (square factors,
8 real flop per complex MAC; device-resident, median of 10): % of the 37.0
TF/s fp64 roofline. python tools/auto_sweep_c.py [lo hi step]"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import paper_2112_11238_b200 as mm  # noqa: E402
from timing import timeit  # noqa: E402

lo, hi, step = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (64, 320, 16)
for n in range(lo, hi + 1, step):
    T = mm.colmajor_empty((n, n, n), torch.complex128, "cuda").normal_()
    Ls = [mm.to_colmajor(torch.randn(n, n, dtype=torch.complex128, device="cuda")) for _ in range(3)]
    ms = timeit(lambda: mm.tucker(T, Ls))
    tf = 3 * 8 * n ** 4 / ms / 1e9
    print(json.dumps({"n": n, "tf": round(tf, 1), "pct": round(100 * tf / 37.0, 1)}), flush=True)
    del T
