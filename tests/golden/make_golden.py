"""Generate the golden vectors in tests/golden/golden.npz.

Inputs are drawn with the reference's generator (std::mt19937_64 + a fresh
std::normal_distribution per object, tools/mumode_cli.cpp:92-121, via
paper_2112_11238_b200.Rng which calls the same libstdc++ code). Outputs are
computed by the REFERENCE LIBRARY ITSELF (oracle/_ref, compiled from
/root/reference/proj/src by oracle/Makefile): ops::tucker, ops::cttucker,
ops::kronsumv, core::mode_product, kronref::kron_apply_oracle, la::expm.

Run in the build container (needs /root/reference only to have built
oracle/_ref):  python tests/golden/make_golden.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle as O  # noqa: E402
from paper_2112_11238_b200 import Rng  # noqa: E402

OUT = Path(__file__).resolve().parent / "golden.npz"


def main():
    data: dict[str, np.ndarray] = {}
    g = Rng(1234)

    def put(key, arr):
        data[key] = np.asarray(arr)

    # validate-suite style cases (tools/mumode_cli.cpp:125-145): d = 1 + g()%5,
    # in/out extents 1 + g()%4, tensor then matrices.
    for c in range(24):
        cplx = c % 2 == 1
        d = 1 + int(g.u64(1)[0] % 5)
        raw = g.u64(2 * d)
        m = [1 + int(raw[2 * k] % 4) for k in range(d)]
        n = [1 + int(raw[2 * k + 1] % 4) for k in range(d)]
        T = g.normal(m, cplx)
        Ls = [g.normal((n[k], m[k]), cplx) for k in range(d)]
        S = O.ref_tucker(T, Ls)
        K = O.ref_tucker(T, Ls, "kron")
        put(f"tk{c}_T", T)
        for k, L in enumerate(Ls):
            put(f"tk{c}_L{k}", L)
        put(f"tk{c}_S", S)
        put(f"tk{c}_K", K)

    # cttucker (complex adjoint): Psi_mu is m x n
    for c in range(6):
        d = 1 + c % 4
        m = [2 + (c + k) % 3 for k in range(d)]
        n = [1 + (2 * c + k) % 4 for k in range(d)]
        T = g.normal(m, True)
        Ps = [g.normal((m[k], n[k]), True) for k in range(d)]
        put(f"ct{c}_T", T)
        for k, P in enumerate(Ps):
            put(f"ct{c}_P{k}", P)
        put(f"ct{c}_S", O.ref_tucker(T, Ps, "cttucker"))

    # mode products on every mode of an order-4 tensor, rectangular factors
    T = g.normal((5, 6, 4, 3))
    put("mp_T", T)
    for mu in range(1, 5):
        L = g.normal((7 - mu, T.shape[mu - 1]))
        put(f"mp_L{mu}", L)
        put(f"mp_S{mu}", O.ref_mode_product(T, L, mu))
    Tc = g.normal((4, 3, 5), True)
    put("mpc_T", Tc)
    for mu in range(1, 4):
        L = g.normal((6, Tc.shape[mu - 1]), True)
        put(f"mpc_L{mu}", L)
        put(f"mpc_S{mu}", O.ref_mode_product(Tc, L, mu))

    # kronsumv
    V = g.normal((4, 5, 3))
    As = [g.normal((e, e)) for e in V.shape]
    put("ks_V", V)
    for k, A in enumerate(As):
        put(f"ks_A{k}", A)
    put("ks_W", O.ref_tucker(V, As, "kronsumv"))

    # promotion: real tensor, complex stack
    T = g.normal((3, 4, 2))
    Ls = [g.normal((2 + k, T.shape[k]), True) for k in range(3)]
    put("pr_T", T)
    for k, L in enumerate(Ls):
        put(f"pr_L{k}", L)
    put("pr_S", O.ref_tucker(T, Ls))

    # scaled configs (same generators as BASELINE configs, small sizes)
    T = g.normal((24, 24, 24))
    Ls = [g.normal((24, 24)) for _ in range(3)]
    put("c2_T", T)
    for k, L in enumerate(Ls):
        put(f"c2_L{k}", L)
    put("c2_S", O.ref_tucker(T, Ls))
    # config 3 (exp integrator): A = Laplacian + 0.5 centred advection, n = 20
    n3 = 20
    A = O.port_advection_diffusion(n3, 0.5)
    E = O.ref_expm(1e-3 * A)
    u0 = g.normal((n3, n3, n3))
    u = u0.copy(order="F")
    for _ in range(10):
        u = O.ref_tucker(u, [E, E, E])
    put("c3_A", A)
    put("c3_E", E)
    put("c3_u0", u0)
    put("c3_u10", u)
    # config 4 (complex rectangular): 8^3 -> 12^3
    T = g.normal((8, 8, 8), True)
    Ls = [g.normal((12, 8), True) for _ in range(3)]
    put("c4_T", T)
    for k, L in enumerate(Ls):
        put(f"c4_L{k}", L)
    put("c4_S", O.ref_tucker(T, Ls))
    # config 5 (6-D): 4^6
    T = g.normal((4,) * 6)
    Ls = [g.normal((4, 4)) for _ in range(6)]
    put("c5_T", T)
    for k, L in enumerate(Ls):
        put(f"c5_L{k}", L)
    put("c5_S", O.ref_tucker(T, Ls))
    np.savez_compressed(OUT, **data)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(data)} arrays)")


if __name__ == "__main__":
    main()
