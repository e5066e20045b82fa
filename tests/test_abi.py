"""C-ABI and host-logic tests that need no GPU.

* libmumode_b200.so loads and exports every entry point include/mumode_gpu.h
  declares (and the ctypes binding covers exactly that set);
* without a GPU the engine refuses to run (no silent CPU fallback);
* the reference-shaped API raises the reference's error types and messages
  before touching the device (errors.hpp, tucker.hpp:67-78,
  mode_product.hpp:66-69, tucker.hpp:211-220);
* host preprocessing: the seeded generator and expm.
"""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import oracle as O
import paper_2112_11238_b200 as mm
from paper_2112_11238_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "mumode_gpu.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mumode_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_are_exported_and_bound():
    so = ctypes.CDLL(str(_lib.LIB_PATH))
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(so, s), f"{s} declared in mumode_gpu.h but not exported"
    assert set(syms) == set(_lib.SIGNATURES), "ctypes binding out of sync with the header"


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
    assert "sm_90" not in out.stdout and "sm_80" not in out.stdout


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    rc = _lib.lib().mumode_handle_create(ctypes.byref(h), 0)
    assert rc == 3  # MUMODE_ERR_CUDA
    assert b"no CPU path" in _lib.lib().mumode_last_error() or b"CUDA" in _lib.lib().mumode_last_error()
    with pytest.raises(mm.CudaError):
        mm.tucker(np.ones((2, 2), order="F"), [np.eye(2), np.eye(2)])


# ---- error contract (raised before any device work) ------------------------

def test_tucker_size_errors_name_the_mode():
    T = np.zeros((2, 3, 4), order="F")
    bad = [np.eye(2), np.zeros((3, 2)), np.eye(4)]
    with pytest.raises(mm.SizeError, match="mode 2"):
        mm.tucker(T, bad)
    with pytest.raises(mm.SizeError):
        mm.tucker(T, [np.eye(2), np.eye(3)])
    with pytest.raises(mm.SizeError, match="mode 3"):
        mm.cttucker(T, [np.eye(2), np.eye(3), np.zeros((3, 4))])


def test_mode_product_errors():
    T = np.zeros((3, 4, 2), order="F")
    L = np.zeros((5, 3))
    with pytest.raises(mm.SizeError, match="mode 2"):
        mm.mode_product(T, L, 2)
    with pytest.raises(mm.ArgumentError):
        mm.mode_product(T, L, 7)
    with pytest.raises(mm.ArgumentError):
        mm.mode_product(T, L, 0)


def test_kronsumv_errors():
    V = np.zeros((2, 3), order="F")
    with pytest.raises(mm.SizeError):
        mm.kronsumv(V, [np.zeros((2, 3)), np.eye(3)])
    with pytest.raises(mm.SizeError, match="mode 2"):
        mm.kronsumv(V, [np.eye(2), np.eye(2)])
    with pytest.raises(mm.SizeError):
        mm.kronsumv(V, [np.eye(2)])


def test_error_types_are_value_errors_like_std_invalid_argument():
    assert issubclass(mm.SizeError, ValueError) and issubclass(mm.ArgumentError, ValueError)


# ---- host preprocessing -----------------------------------------------------

def test_rng_engine_known_answer():
    # C++ [rand.predef]: the 10000th consecutive invocation of a
    # default-constructed mt19937_64 (seed 5489) produces 9981545732273789042.
    r = mm.Rng(5489)
    assert int(r.u64(10000)[-1]) == 9981545732273789042


def test_rng_fresh_distribution_per_object():
    # two fills from one engine == one engine stream consumed in order, with a
    # fresh distribution for each object (polar pairs are not shared)
    a = mm.Rng(1234)
    x = a.normal((3,))
    y = a.normal((4,))
    b = mm.Rng(1234)
    x2 = b.normal((3,))
    y2 = b.normal((4,))
    np.testing.assert_array_equal(x, x2)
    np.testing.assert_array_equal(y, y2)
    c = mm.Rng(1234)
    xy = c.normal((7,))
    np.testing.assert_array_equal(xy[:3], x)  # the first object's draws match
    assert not np.array_equal(xy[3:], y)      # the discarded cached sample shifts the rest


def test_rng_matches_golden_inputs():
    # the golden inputs were drawn by the same generator: re-draw the first case
    gold = np.load(ROOT / "tests" / "golden" / "golden.npz")
    g = mm.Rng(1234)
    d = 1 + int(g.u64(1)[0] % 5)
    raw = g.u64(2 * d)
    m = [1 + int(raw[2 * k] % 4) for k in range(d)]
    T = g.normal(m, False)
    np.testing.assert_array_equal(T, gold["tk0_T"])


def test_expm_matches_reference_expm():
    # the host expm reproduces la::expm (src/expm.cpp:97-151) bit for bit:
    # k-ordered FMA products like cblas_dgemm, lu_factor's reciprocal-pivot
    # elimination, and cblas_dtrsm's 16-row-block solve order (n <= 384)
    gold = np.load(ROOT / "tests" / "golden" / "golden.npz")
    A = gold["c3_A"]
    E = mm.expm(1e-3 * A)
    np.testing.assert_array_equal(E, gold["c3_E"])
    # every Pade branch (degrees 3..13, with and without squaring), sizes
    # around the 16-row blocks of the triangular solves
    rng = np.random.default_rng(3)
    for n in (1, 6, 16, 17, 37, 128, 200, 255):
        for scale in (1e-6, 1e-3, 0.2, 1.0, 3.0, 40.0 / n):
            B = np.asfortranarray(rng.standard_normal((n, n)) * scale)
            got = mm.expm(B)
            if O.ref_available():
                np.testing.assert_array_equal(got, O.ref_expm(B), err_msg=f"n={n} scale={scale}")
    np.testing.assert_array_equal(mm.expm(np.zeros((3, 3))), np.eye(3))


def test_factorized_stack_refuses_singular_matrices():
    # test_tucker_ops.cpp:285-288 (host factorization, no GPU needed)
    with pytest.raises(mm.NumericalError, match="singular pivot"):
        mm.FactorizedStack([np.zeros((2, 2))])
    with pytest.raises(mm.SizeError, match="square"):
        mm.FactorizedStack([np.zeros((2, 3))])
    P = np.array([[4.0, 1.0], [2.0, 3.0]])
    F = mm.FactorizedStack([P])
    lu, piv = F.factor(1)
    L = np.tril(lu, -1) + np.eye(2)
    U = np.triu(lu)
    np.testing.assert_allclose(L @ U, P[[0, 1]], atol=1e-15)
    assert list(piv) == [0, 1]


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built")
def test_lu_factor_bitwise_equals_reference():
    # FactorizedStack<T> holds la::lu_factor's factors (lu.hpp:23-47) bit for bit,
    # real and complex, including pivoting on ill-conditioned matrices
    rng = np.random.default_rng(3)
    for n in [1, 2, 3, 8, 24, 40, 97, 200]:
        for cplx in (False, True):
            P = rng.standard_normal((n, n))
            if cplx:
                P = P + 1j * rng.standard_normal((n, n))
            U, _, Vt = np.linalg.svd(P)
            P = np.asfortranarray((U * np.logspace(0, -9, n)) @ Vt)
            lu, piv = O.ref_lu_factor(P)
            F = mm.FactorizedStack([P])
            np.testing.assert_array_equal(F.lu[0], lu)
            np.testing.assert_array_equal(F.piv[0], piv)
            assert F.cplx == cplx


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built")
def test_symtridiag_eig_bitwise_equals_reference():
    # la::symtridiag_eig with FullVectors (src/tridiag.cpp:12-90): the direct
    # solver's eigenpairs are the reference's, bit for bit
    rng = np.random.default_rng(4)
    for n in [1, 2, 3, 10, 64, 200, 257]:
        d, e = rng.standard_normal(n), rng.standard_normal(n - 1)
        w, V = mm.symtridiag_eig(d, e)
        wr, Vr = O.ref_symtridiag_eig(d, e)
        np.testing.assert_array_equal(w, wr)
        np.testing.assert_array_equal(V, Vr)
    # the IMEX factor M = I/d - tau A of the Dirichlet Laplacian (imex.cpp:108-112)
    A = O.ref_laplacian(200)
    M = np.eye(200) / 3 + (-1e-3) * A
    w, V = mm.symtridiag_eig(*mm.extract_tridiag(M))
    wr, Vr = O.ref_symtridiag_eig(np.diag(M).copy(), 0.5 * (np.diag(M, 1) + np.diag(M, -1)))
    np.testing.assert_array_equal(w, wr)
    np.testing.assert_array_equal(V, Vr)


def test_extract_tridiag_rejects_like_reference():
    # src/imex.cpp:28-48: entries off the three diagonals, or an asymmetric
    # off-diagonal pair beyond 1e-12 of the largest entry, are ArgumentErrors
    A = np.eye(5)
    A[0, 3] = 1e-300
    with pytest.raises(mm.ArgumentError, match="not tridiagonal"):
        mm.extract_tridiag(A)
    A = np.diag(np.ones(4)) + np.diag(np.ones(3), 1)
    with pytest.raises(mm.ArgumentError, match="not symmetric"):
        mm.extract_tridiag(A)
    with pytest.raises(mm.ArgumentError, match="not symmetric"):
        mm.KronSumSolver(Ms=[A, A])
    B = np.diag(np.full(4, 2.0)) + np.diag(np.full(3, 1.0), 1) + np.diag(np.full(3, 1.0 + 1e-14), -1)
    d, e = mm.extract_tridiag(B)  # within the 1e-12 relative tolerance: averaged
    np.testing.assert_array_equal(d, np.full(4, 2.0))
    np.testing.assert_array_equal(e, np.full(3, 0.5 * (1.0 + (1.0 + 1e-14))))
    with pytest.raises(mm.ArgumentError, match="fewer than diag"):
        mm.symtridiag_eig(np.ones(3), np.ones(3))


def test_empty_tensors_rejected_like_reference():
    # Shape({2, 0, 3}) and Shape({}) throw ArgumentError (test_tensor_core.cpp:17-20);
    # the engine rejects them before touching a device, at both layers
    with pytest.raises(mm.ArgumentError, match="extents must be positive"):
        mm.tucker(np.zeros((2, 0, 3), order="F"), [np.eye(2), np.zeros((1, 0)), np.eye(3)])
    with pytest.raises(mm.ArgumentError, match="order must be >= 1"):
        mm.mode_product(np.zeros(()), np.eye(1), 1)
    from paper_2112_11238_b200.dist import slab_plan_offsets
    with pytest.raises(mm.ArgumentError, match="extents must be positive"):
        slab_plan_offsets(1, (2, 0, 3), (2, 1, 3))


def test_matricize_mode_action_tuckerfun_host_helpers():
    # matricize.hpp / mode_product.hpp:88-100 / tucker.hpp:169-185 semantics
    rng = np.random.default_rng(11)
    T = np.asfortranarray(rng.standard_normal((3, 4, 5)))
    for mu in (1, 2, 3):
        M = mm.matricize(T, mu)
        assert M.shape == (T.shape[mu - 1], T.size // T.shape[mu - 1])
        np.testing.assert_array_equal(mm.dematricize(M, mu, T.shape), T)
    # column order: remaining indices, earliest fastest (test_tensor_core.cpp)
    M2 = mm.matricize(T, 2)
    assert M2[3, 1 + 3 * 4] == T[1, 3, 4]
    Ls = [rng.standard_normal((2, 3)), rng.standard_normal((6, 4)), rng.standard_normal((5, 5))]
    ops = [(L.shape[0], (lambda L: (lambda X: L @ X))(L)) for L in Ls]
    ref = O.port_tucker(T, Ls)
    assert O.rel_max(mm.tuckerfun(T, ops), ref) < 1e-13
    assert O.rel_max(mm.mode_action(T, ops[1][1], 2), O.port_mode_product(T, Ls[1], 2)) < 1e-13
    with pytest.raises(mm.ContractError, match="mode 3"):
        mm.tuckerfun(T, ops[:2] + [(4, ops[2][1])])
    with pytest.raises(mm.ContractError):
        mm.mode_action(T, lambda X: X[:, :-1], 1)
