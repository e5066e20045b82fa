"""Parity report: the CUDA path vs the compiled reference library (oracle/_ref)
on the BASELINE configs, identical seeded bytes. Prints one JSON object with
relative Frobenius and relative max-norm errors per config and PASS / FAIL
against the north-star gate (relative Frobenius <= 1e-12); exit status 1 on
any FAIL. --inject-fault perturbs one element of the C2 result (the
reference CLI's test-only flag, tools/mumode_cli.cpp:142,168) so the failure
path is exercised. Test infrastructure: imports the oracle as the checker."""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle as O  # noqa: E402
import paper_2112_11238_b200 as mm  # noqa: E402


def dev(x):
    return torch.from_numpy(np.asfortranarray(x)).cuda()


def host(t):
    return t.cpu().numpy()


GATE = 1e-12
INJECT = False


def rec(out, name, got, want, t_ref):
    if INJECT and name == "C2_tucker_256":
        got = got.copy()
        got[(0,) * got.ndim] += 1e-6 * float(np.max(np.abs(want)))
    err = O.rel_fro(got, want)
    out[name] = {"rel_fro": err, "rel_max": O.rel_max(got, want), "ref_seconds": round(t_ref, 3),
                 "status": "PASS" if err <= GATE else "FAIL"}


def main():
    global INJECT
    ap = argparse.ArgumentParser()
    ap.add_argument("--inject-fault", action="store_true",
                    help="test-only: corrupt the C2 result to exercise the failure path")
    ap.add_argument("--quick", action="store_true", help="C1 and C2 only")
    args = ap.parse_args()
    INJECT = args.inject_fault
    out = {"reference": f"oracle/_ref (reference library), OpenBLAS {O.ref_blas_kernel_name()}"}
    g = mm.Rng(1234 + 100)
    L1, L2 = g.normal((100, 100)), g.normal((100, 100))
    T = g.normal((100, 100))
    t0 = time.time(); ref = O.ref_tucker(T, [L1, L2]); t = time.time() - t0
    rec(out, "C1_2d_n100", host(mm.tucker(dev(T), [dev(L1), dev(L2)])), ref, t)

    g = mm.Rng(1234)
    T = g.normal((256,) * 3)
    Ls = [g.normal((256, 256)) for _ in range(3)]
    t0 = time.time(); ref = O.ref_tucker(T, Ls); t = time.time() - t0
    rec(out, "C2_tucker_256", host(mm.tucker(dev(T), [dev(L) for L in Ls])), ref, t)
    for mu in (1, 2, 3):
        t0 = time.time(); ref = O.ref_mode_product(T, Ls[mu - 1], mu); t = time.time() - t0
        rec(out, f"C2_mode{mu}", host(mm.mode_product(dev(T), dev(Ls[mu - 1]), mu)), ref, t)
    if args.quick:
        return finish(out)

    n = 200
    A = O.port_advection_diffusion(n, 0.5)
    E = O.ref_expm(1e-3 * A)
    g = mm.Rng(1234)
    u0 = g.normal((n,) * 3)
    t0 = time.time()
    u = u0
    steps = []
    for s in range(100):
        u = O.ref_tucker(u, [E, E, E])
        if s in (0, 9, 99):
            steps.append((s + 1, u))
    t = time.time() - t0
    for k, uref in steps:
        rec(out, f"C3_expint_step{k}_sameE", host(mm.expint(dev(u0), [dev(E)] * 3, k)), uref, t)
    E2 = mm.expm(1e-3 * A)
    out["C3_expm_engine_vs_reference"] = O.rel_fro(E2, E)
    rec(out, "C3_expint_step100_engineE", host(mm.expint(dev(u0), [dev(E2)] * 3, 100)), steps[-1][1], t)

    g = mm.Rng(1234)
    T = g.normal((128,) * 3, True)
    Ls = [g.normal((192, 128), True) for _ in range(3)]
    t0 = time.time(); ref = O.ref_tucker(T, Ls); t = time.time() - t0
    rec(out, "C4_complex_128_to_192", host(mm.tucker(dev(T), [dev(L) for L in Ls])), ref, t)

    g = mm.Rng(1234)
    T = g.normal((24,) * 6)
    Ls = [g.normal((24, 24)) for _ in range(6)]
    t0 = time.time(); ref = O.ref_tucker(T, Ls); t = time.time() - t0
    rec(out, "C5_6d_24", host(mm.tucker(dev(T), [dev(L) for L in Ls])), ref, t)
    return finish(out)


def finish(out) -> int:
    bad = [k for k, v in out.items() if isinstance(v, dict) and v.get("status") == "FAIL"]
    out["overall"] = "FAIL" if bad else "PASS"
    out["failed"] = bad
    print(json.dumps(out, indent=1))
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
