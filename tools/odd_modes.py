"""Per-mode timing of the ragged shapes the padded odd-extent chain runs
(mode 1 padded even; later modes with ragged K / N), by kernel policy."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in evs)[reps // 2]


if __name__ == "__main__":
    h = mm.get_handle(0)
    for shape in [(256, 255, 255), (202, 201, 201), (256, 256, 256), (200, 200, 200)]:
        T = mm.colmajor_empty(shape, torch.float64, "cuda").normal_()
        for mu in (1, 2, 3):
            e = shape[mu - 1]
            L = mm.to_colmajor(torch.randn(e, e, dtype=torch.float64, device="cuda"))
            row = {"shape": shape, "mu": mu}
            for pol in (0, 8, 3, 4, 5, 6):
                h.set_kernel_policy(pol)
                try:
                    ms = timeit(lambda: mm.mode_product(T, L, mu))
                    row[f"p{pol}"] = round(2 * e * T.numel() / ms / 1e9, 1)
                except Exception as ex:  # noqa: BLE001
                    row[f"p{pol}"] = str(ex)[:30]
            h.set_kernel_policy(0)
            print(json.dumps(row))
