"""`mumode validate --suite tucker` of the reference CLI
(/root/reference/proj/tools/mumode_cli.cpp:125-160) against the B200 engine:
100 real and 100 complex random Tucker cases (order 1..5, extents 1..4, the
reference's draw sequence from std::mt19937_64(seed)) through the engine's
device path, each checked against the reference library's explicit-Kronecker
oracle (kronref::kron_apply_oracle, oracle/_ref) at 1e-13.

--inject-fault corrupts the first real case (S[0] += 1e-6), exactly like the
reference's test-only flag, so the failure path is exercised: the report
says FAIL and the exit status is 1 (the negative control,
tests/test_negative_control.py). Test infrastructure: the oracle is the
checker.
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle as O  # noqa: E402
import paper_2112_11238_b200 as mm  # noqa: E402


def case(g: mm.Rng, cplx: bool, inject: bool) -> float:
    import torch
    d = 1 + int(g.u64(1)[0] % 5)
    ins, outs = [], []
    for _ in range(d):
        ins.append(1 + int(g.u64(1)[0] % 4))
        outs.append(1 + int(g.u64(1)[0] % 4))
    T = g.normal(ins, complex_=cplx)
    Ls = [g.normal((outs[k], ins[k]), complex_=cplx) for k in range(d)]
    fast = mm.tucker(torch.from_numpy(T).cuda(), [torch.from_numpy(L).cuda() for L in Ls]).cpu().numpy()
    if inject:
        fast[(0,) * fast.ndim] += 1e-6
    slow = O.ref_tucker(T, Ls, "kron")
    return float(np.max(np.abs(fast - slow)) / max(float(np.max(np.abs(slow))), 1e-300))


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--seed", type=int, default=1234)
    ap.add_argument("--cases", type=int, default=100)
    ap.add_argument("--inject-fault", action="store_true",
                    help="test-only: corrupt one case to exercise the failure path")
    args = ap.parse_args()
    g = mm.Rng(args.seed)
    worst = 0.0
    for c in range(args.cases):
        worst = max(worst, case(g, False, args.inject_fault and c == 0))
        worst = max(worst, case(g, True, False))
    ok = worst < 1e-13
    print(f"{'tucker-vs-kron-oracle':<24} {'PASS' if ok else 'FAIL'}   worst error {worst:.3e}")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
