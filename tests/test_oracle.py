"""Pin the oracles before trusting them (CPU only, no GPU).

* the plain-C restatement (oracle/liboracle.so) against the golden vectors the
  reference library produced (tests/golden/golden.npz, make_golden.py);
* the restatement against the compiled reference (oracle/_ref) on fresh
  seeded cases, when oracle/_ref is built;
* the reference's own known-answer tests for this path.
"""
from pathlib import Path

import numpy as np
import pytest

import oracle as O

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "golden.npz")


def stack(prefix, tag, d):
    return [GOLD[f"{prefix}_{tag}{k}"] for k in range(d)]


def test_port_matches_golden_tucker_cases():
    # tests the validate-suite cases (tools/mumode_cli.cpp:125-145)
    worst = 0.0
    for c in range(24):
        T = GOLD[f"tk{c}_T"]
        Ls = stack(f"tk{c}", "L", T.ndim)
        S = O.port_tucker(T, Ls)
        worst = max(worst, O.rel_max(S, GOLD[f"tk{c}_S"]), O.rel_max(S, GOLD[f"tk{c}_K"]))
    assert worst < 1e-13


def test_port_matches_golden_cttucker():
    for c in range(6):
        T = GOLD[f"ct{c}_T"]
        Ps = stack(f"ct{c}", "P", T.ndim)
        assert O.rel_max(O.port_tucker(T, Ps, adjoint=True), GOLD[f"ct{c}_S"]) < 1e-14


def test_port_matches_golden_mode_products():
    T = GOLD["mp_T"]
    for mu in range(1, 5):
        S = O.port_mode_product(T, GOLD[f"mp_L{mu}"], mu)
        assert O.rel_max(S, GOLD[f"mp_S{mu}"]) < 1e-13
    Tc = GOLD["mpc_T"]
    for mu in range(1, 4):
        S = O.port_mode_product(Tc, GOLD[f"mpc_L{mu}"], mu)
        assert O.rel_max(S, GOLD[f"mpc_S{mu}"]) < 1e-13


def test_port_matches_golden_kronsumv_and_promotion():
    V = GOLD["ks_V"]
    assert O.rel_max(O.port_kronsumv(V, stack("ks", "A", 3)), GOLD["ks_W"]) < 1e-13
    T = GOLD["pr_T"]
    assert O.rel_max(O.port_tucker(T, stack("pr", "L", 3)), GOLD["pr_S"]) < 1e-15


def test_port_matches_golden_configs():
    assert O.rel_fro(O.port_tucker(GOLD["c2_T"], stack("c2", "L", 3)), GOLD["c2_S"]) < 1e-14
    E = GOLD["c3_E"]
    u = GOLD["c3_u0"]
    for _ in range(10):
        u = O.port_tucker(u, [E, E, E])
    assert O.rel_fro(u, GOLD["c3_u10"]) < 1e-13
    assert O.rel_fro(O.port_tucker(GOLD["c4_T"], stack("c4", "L", 3)), GOLD["c4_S"]) < 1e-14
    assert O.rel_fro(O.port_tucker(GOLD["c5_T"], stack("c5", "L", 6)), GOLD["c5_S"]) < 1e-14
    # the config-3 operator restatement equals the reference stencil + advection
    if O.ref_available():
        n = GOLD["c3_A"].shape[0]
        lap = O.ref_laplacian(n)
        adv = GOLD["c3_A"] - lap
        h = 1.0 / (n + 1)
        assert np.allclose(np.diag(adv, 1), 0.5 / (2 * h)) and np.allclose(np.diag(adv, -1), -0.5 / (2 * h))
    np.testing.assert_array_equal(O.port_advection_diffusion(GOLD["c3_A"].shape[0], 0.5), GOLD["c3_A"])


# ---- known-answer tests of the reference suite (no GPU) -------------------

def test_known_answer_identity_stack_is_exact():
    # test_tucker_ops.cpp:41-52
    rng = np.random.default_rng(100)
    for _ in range(10):
        d = int(rng.integers(1, 6))
        m = [int(x) for x in rng.integers(1, 5, d)]
        T = np.asfortranarray(rng.uniform(-1, 1, m))
        S = O.port_tucker(T, [np.eye(e) for e in m])
        assert np.max(np.abs(S - T)) == 0.0


def test_known_answer_cttucker_scalar():
    # test_tucker_ops.cpp:208-215: Psi = i, T = 2 + i -> S = -i * T
    T = np.array([2.0 + 1.0j])
    S = O.port_tucker(T, [np.array([[1.0j]])], adjoint=True)
    assert abs(S[0] - (-1.0j) * T[0]) < 1e-15


def test_known_answer_kronsumv_identity_is_3v():
    # test_tucker_ops.cpp:290-300
    V = np.asfortranarray(np.random.default_rng(117).uniform(-1, 1, (2, 3, 2)))
    W = O.port_kronsumv(V, [np.eye(2), np.eye(3), np.eye(2)])
    assert np.max(np.abs(W - 3.0 * V)) == 0.0


def test_known_answer_permute_remap():
    # test_tensor_core.cpp "order 3 remap oracle"
    T = np.asfortranarray(np.arange(24, dtype=float).reshape((2, 3, 4), order="F"))
    S = O.port_permute(T, [3, 1, 2])
    assert S.shape == (4, 2, 3)
    for j1 in range(2):
        for j2 in range(3):
            for j3 in range(4):
                assert S[j3, j1, j2] == T[j1, j2, j3]


# ---- restatement vs the compiled reference on fresh seeded cases ----------

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@needs_ref
def test_port_vs_ref_random_orders_1_to_5():
    rng = np.random.default_rng(102)
    worst = 0.0
    for rep in range(60):
        d = int(rng.integers(1, 6))
        m = [int(x) for x in rng.integers(1, 5, d)]
        n = [int(x) for x in rng.integers(1, 5, d)]
        cplx = rep % 2 == 1
        T = rng.uniform(-1, 1, m) + (1j * rng.uniform(-1, 1, m) if cplx else 0)
        Ls = [rng.uniform(-1, 1, (n[k], m[k])) + (1j * rng.uniform(-1, 1, (n[k], m[k])) if cplx else 0)
              for k in range(d)]
        worst = max(worst, O.rel_max(O.port_tucker(T, Ls), O.ref_tucker(T, Ls)))
    assert worst < 1e-13


@needs_ref
def test_port_vs_ref_mode_product_loops_oracle():
    # test_tensor_core.cpp:207-223 (nested-loop oracle, <= 200 elements)
    rng = np.random.default_rng(19)
    done = 0
    while done < 60:
        d = int(rng.integers(1, 6))
        m = [int(x) for x in rng.integers(1, 6, d)]
        if int(np.prod(m)) > 200:
            continue
        done += 1
        mu = int(rng.integers(1, d + 1))
        L = rng.uniform(-1, 1, (int(rng.integers(1, 6)), m[mu - 1]))
        T = rng.uniform(-1, 1, m)
        a = O.port_mode_product(T, L, mu)
        assert O.rel_max(a, O.ref_mode_product(T, L, mu, loops=True)) < 1e-13
        assert O.rel_max(a, O.ref_mode_product(T, L, mu)) < 1e-13


@needs_ref
def test_ref_size_error_names_mode():
    T = np.zeros((2, 3, 4), order="F")
    bad = [np.eye(2), np.zeros((3, 2)), np.eye(4)]
    with pytest.raises(O.RefError) as e:
        O.ref_tucker(T, bad)
    assert e.value.code == 1 and "mode 2" in str(e.value)


def test_rel_metrics():
    a = np.array([1.0, 2.0])
    assert O.rel_max(a, a) == 0.0 and O.rel_fro(a, a) == 0.0
    assert abs(O.rel_fro(a * (1 + 1e-12), a) - 1e-12) < 1e-15
