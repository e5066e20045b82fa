"""Short runs of one configuration for ncu (`ncu ... python tools/prof.py c5`):
a few warm-up applications, then one more; nothing is timed here.

  c2        3-D Tucker 256^3 (BASELINE configs[1])
  c3        3-D Tucker 200^3 with a contraction-like factor (configs[2] step)
  c4        complex 128^3 -> 192^3 (configs[3])
  c5        6-D 24^6 (configs[4])
  d6 N      6-D N^6 (the paper's d = 6 sizes, e.g. 18, 20)
  --policy P  run under kernel policy P (e.g. 16: in-place block passes)
  kronsumv  Kronecker-sum action at 24^6 and 200^3
  itucker   inverse Tucker 200^3
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402


def normal(shape, cplx=False):
    return mm.colmajor_empty(shape, torch.complex128 if cplx else torch.float64, "cuda").normal_()


def mats(ns, ms, cplx=False):
    dt = torch.complex128 if cplx else torch.float64
    return [mm.to_colmajor(torch.randn(n, m, dtype=dt, device="cuda")) for n, m in zip(ns, ms)]


def run(fn, reps=3):
    for _ in range(reps + 1):
        out = fn()
    torch.cuda.synchronize()
    print("ok", float(out.abs().max()))


def main():
    if "--policy" in sys.argv:  # kernel policy for the run (mumode_set_kernel_policy)
        i = sys.argv.index("--policy")
        mm.get_handle(0).set_kernel_policy(int(sys.argv[i + 1]))
        del sys.argv[i:i + 2]
    what = sys.argv[1]
    if what == "c2":
        T, Ls = normal((256,) * 3), mats((256,) * 3, (256,) * 3)
        run(lambda: mm.tucker(T, Ls))
    elif what == "c3":
        T = normal((200,) * 3)
        E = [mm.to_colmajor(torch.randn(200, 200, dtype=torch.float64, device="cuda") * 0.07)] * 3
        run(lambda: mm.tucker(T, E))
    elif what == "c4":
        T, Ls = normal((128,) * 3, True), mats((192,) * 3, (128,) * 3, True)
        run(lambda: mm.tucker(T, Ls))
    elif what == "c5":
        T, Ls = normal((24,) * 6), mats((24,) * 6, (24,) * 6)
        run(lambda: mm.tucker(T, Ls))
    elif what == "d6":
        n = int(sys.argv[2])
        T, Ls = normal((n,) * 6), mats((n,) * 6, (n,) * 6)
        run(lambda: mm.tucker(T, Ls))
    elif what == "kronsumv":
        for n, d in ((24, 6), (200, 3)):
            V, As = normal((n,) * d), mats((n,) * d, (n,) * d)
            run(lambda: mm.kronsumv(V, As), reps=2)
    elif what == "itucker":
        T = normal((200,) * 3)
        F = mm.FactorizedStack([np.random.default_rng(k).standard_normal((200, 200)) + 20 * np.eye(200)
                                for k in range(3)])
        run(lambda: mm.itucker(T, F), reps=2)
    else:
        raise SystemExit(__doc__)


if __name__ == "__main__":
    main()
