"""C4 (complex 128^3 -> 192^3) timing per mode and for the Tucker chain under
auto and each forced complex tile configuration (development aid; bench.py is
the contract). 8 real flops per complex MAC."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402
from quick_bench import timeit  # noqa: E402


def main():
    h = mm.get_handle(0)
    T = mm.colmajor_empty((128,) * 3, torch.complex128, "cuda").normal_()
    Ls = [mm.to_colmajor(torch.randn(192, 128, dtype=torch.complex128, device="cuda")) for _ in range(3)]
    for policy in (0, 4, 5, 6, 7):
        h.set_kernel_policy(policy)
        row = {"policy": policy}
        cur, ext = T, [128, 128, 128]
        for mu in (1, 2, 3):
            src = cur
            ms = timeit(lambda: mm.mode_product(src, Ls[mu - 1], mu), reps=20)
            numel = ext[0] * ext[1] * ext[2]
            row[f"mode{mu}_ms"] = round(ms, 4)
            row[f"mode{mu}_tf"] = round(8.0 * 192 * numel / ms / 1e9, 2)
            cur = mm.mode_product(src, Ls[mu - 1], mu)
            ext[mu - 1] = 192
        ms = timeit(lambda: mm.tucker(T, Ls), reps=20)
        row["tucker_ms"] = round(ms, 4)
        row["tucker_tf"] = round(1.530e10 / ms / 1e9, 2)
        print(json.dumps(row), flush=True)
    h.set_kernel_policy(0)


if __name__ == "__main__":
    main()
