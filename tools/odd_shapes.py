"""Timing of Tucker on shapes the TMA path cannot describe (odd leading
extents -> 8-byte-aligned strides) vs nearby even shapes."""
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


for n in (255, 256, 201, 200, 129):
    T = mm.colmajor_empty((n, n, n), torch.float64, "cuda").normal_()
    Ls = [mm.to_colmajor(torch.randn(n, n, dtype=torch.float64, device="cuda")) for _ in range(3)]
    ms = timeit(lambda: mm.tucker(T, Ls))
    print(json.dumps({"n": n, "tucker_ms": round(ms, 4), "tflops": round(3 * 2 * n ** 4 / ms / 1e9, 2)}))

# complex: odd extents (SIMT generic kernel today) vs even (TMA/DMMA)
for m, nn in ((127, 191), (128, 192), (99, 101)):
    T = mm.colmajor_empty((m, m, m), torch.complex128, "cuda")
    T.real.normal_()
    T.imag.normal_()
    Ls = [mm.to_colmajor(torch.randn(nn, m, dtype=torch.complex128, device="cuda")) for _ in range(3)]
    ms = timeit(lambda: mm.tucker(T, Ls))
    fl = 8 * (nn * m ** 3 + nn * nn * m ** 2 + nn ** 3 * m)
    print(json.dumps({"complex": [m, nn], "tucker_ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 2)}))
