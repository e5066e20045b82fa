"""Time the fused two-mode passes of C5 (24^6) and of a few other small-mode
shapes under several kernel policies (0 = auto: warp-specialised passes,
12 = the non-warp-specialised kernels, 9 / 10 = tail pass forced / off), and
check every policy's outputs are bitwise equal to the first one's.
argv: policies (e.g. 0,12) and shapes (e.g. 24x24x24x24x24x24)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402
from paper_2112_11238_b200 import _lib  # noqa: E402

lib = _lib.lib()
h = mm.get_handle(0)
h.bind_torch_stream()
variants = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 12]
shapes = [tuple(int(x) for x in s.split("x")) for s in sys.argv[2].split(",")] if len(sys.argv) > 2 else \
    [(24,) * 6, (16,) * 6, (8,) * 8, (24,) * 4, (24, 24, 24, 24, 24)]
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")


def run_range(T, Ls, S, shape, lo, hi):
    P = _lib.ptr_array([L.data_ptr() for L in Ls])
    m = _lib.i64_array(shape)
    rc = lib.mumode_tucker_range_f64(h.h, len(shape), m, m, T.data_ptr(), P, S.data_ptr(), lo, hi)
    assert rc == 0, lib.mumode_last_error().decode()


def timed(fn, reps=8):
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2] * 1e3


for shape in shapes:
    torch.manual_seed(0)
    T = mm.colmajor_empty(shape, torch.float64, "cuda").normal_()
    Ls = [mm.to_colmajor(torch.randn(s, s, dtype=torch.float64, device="cuda")) for s in shape]
    d = len(shape)
    ref = {}
    for v in variants:
        h.set_kernel_policy(v)
        line = [f"{'x'.join(map(str, shape))} policy {v}:"]
        for lo in range(1, d, 2):
            S = torch.empty_like(T)
            us = timed(lambda: run_range(T, Ls, S, shape, lo, lo + 1))
            run_range(T, Ls, S, shape, lo, lo + 1)
            torch.cuda.synchronize()
            key = lo
            if v == variants[0]:
                ref[key] = S.clone()
                ok = "ref"
            else:
                ok = "bitwise" if torch.equal(S, ref[key]) else f"DIFF {float((S - ref[key]).abs().max()):.3e}"
            line.append(f"({lo},{lo + 1}) {us:.1f} us {ok}")
        S = torch.empty_like(T)
        us = timed(lambda: mm.tucker(T, Ls), reps=5)
        line.append(f"tucker {us:.1f} us")
        print("  ".join(line), flush=True)
h.set_kernel_policy(0)
