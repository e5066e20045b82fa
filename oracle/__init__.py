"""CPU oracles for the mu-mode product / Tucker hot path.

TEST INFRASTRUCTURE ONLY. This package may be imported by ``tests/``,
``__graft_entry__.smoke()`` (as the checker) and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py``. The product package
``paper_2112_11238_b200`` never imports it, and nothing here is ever the thing
measured as "our" throughput.

Two oracles:

* ``port``  -- ``liboracle.so``, a plain-C restatement of the reference's
  algorithm (``oracle/mumode_oracle.c``, each function citing the reference
  file:line it follows).
* ``ref``   -- ``_ref/libmumode_ref.so``, the reference library itself compiled
  from ``/root/reference/proj/src/*.cpp`` by ``oracle/Makefile`` and called
  through ``oracle/ref_shim.cpp``. It runs the reference's own OpenMP +
  OpenBLAS code path.

All arrays are numpy, column-major (Fortran order) float64 or complex128,
matching ``proj/include/mumode/shape.hpp:68-77``.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libmumode_ref.so"

_port = None
_ref = None

I64P = ctypes.POINTER(ctypes.c_int64)
DP = ctypes.POINTER(ctypes.c_double)


def _cpu_coretype() -> str | None:
    """Mirror of the reference's core-type steering (src/gemm.cpp:21-38): with a
    shared OpenBLAS the reference's own constructor runs too late, so it is set
    here before the library is loaded."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    if " avx512f" in line:
                        return "SKYLAKEX"
                    if " avx2" in line:
                        return "HASWELL"
                    return None
    except OSError:
        return None
    return None


def port_lib():
    global _port
    if _port is None:
        if not PORT_SO.exists():
            raise RuntimeError(f"oracle port not built: {PORT_SO} (run `make -C oracle`)")
        _port = ctypes.CDLL(str(PORT_SO), mode=ctypes.RTLD_LOCAL)
        _port.orc_tucker.restype = ctypes.c_int
    return _port


def ref_available() -> bool:
    return REF_SO.exists()


def ref_lib(threads: int | None = None):
    """Load the compiled reference. `threads` sets OMP/OpenBLAS threads (all
    host cores by default) -- only effective before the first load."""
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            raise RuntimeError(f"reference oracle not built: {REF_SO} (run `make -C oracle ref`)")
        n = str(threads or os.cpu_count() or 1)
        os.environ.setdefault("OMP_NUM_THREADS", n)
        os.environ.setdefault("OPENBLAS_NUM_THREADS", n)
        ct = _cpu_coretype()
        if ct:
            os.environ.setdefault("OPENBLAS_CORETYPE", ct)
        _ref = ctypes.CDLL(str(REF_SO), mode=ctypes.RTLD_LOCAL)
        _ref.ref_last_error.restype = ctypes.c_char_p
        _ref.ref_blas_kernel_name.restype = ctypes.c_char_p
    return _ref


class RefError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


_REF_ERR = {1: "SizeError", 2: "ArgumentError", 6: "ContractError", 7: "NumericalError"}


def _check(rc: int):
    if rc != 0:
        msg = _ref.ref_last_error().decode()
        raise RefError(rc, f"{_REF_ERR.get(rc, 'Error')}: {msg}")


def _i64(vals) -> ctypes.Array:
    return (ctypes.c_int64 * len(vals))(*[int(v) for v in vals])


def _f(a: np.ndarray, cplx: bool) -> np.ndarray:
    return np.asfortranarray(a, dtype=np.complex128 if cplx else np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(DP)


def _ptrs(mats):
    arr = (DP * len(mats))()
    for i, m in enumerate(mats):
        arr[i] = _ptr(m)
    return arr


# ----------------------------------------------------------------- port (C)

def port_mode_product(T: np.ndarray, L: np.ndarray, mu: int, adjoint: bool = False) -> np.ndarray:
    cplx = np.iscomplexobj(T) or np.iscomplexobj(L)
    T = _f(T, cplx)
    L = _f(L, cplx)
    m = list(T.shape)
    n = L.shape[1] if adjoint else L.shape[0]
    out = list(m)
    out[mu - 1] = n
    S = np.empty(out, dtype=T.dtype, order="F")
    fn = port_lib().orc_mode_product_c128 if cplx else port_lib().orc_mode_product_f64
    fn(ctypes.c_int(T.ndim), _i64(m), ctypes.c_int(mu), ctypes.c_int64(n), _ptr(T), _ptr(L),
       ctypes.c_int64(L.shape[0]), ctypes.c_int(int(adjoint)), _ptr(S))
    return S


def port_tucker(T: np.ndarray, Ls, adjoint: bool = False) -> np.ndarray:
    cplx = np.iscomplexobj(T) or any(np.iscomplexobj(L) for L in Ls)
    T = _f(T, cplx)
    Ls = [_f(L, cplx) for L in Ls]
    d = T.ndim
    n = [L.shape[1] if adjoint else L.shape[0] for L in Ls]
    S = np.empty(n, dtype=T.dtype, order="F")
    rc = port_lib().orc_tucker(ctypes.c_int(2 if cplx else 1), ctypes.c_int(d), _i64(T.shape),
                               _i64(n), _ptr(T), _ptrs(Ls), _i64([L.shape[0] for L in Ls]),
                               ctypes.c_int(int(adjoint)), _ptr(S))
    if rc != 0:
        raise ValueError("orc_tucker failed")
    return S


def port_kronsumv(V: np.ndarray, As) -> np.ndarray:
    V = _f(V, False)
    As = [_f(A, False) for A in As]
    W = np.empty(V.shape, order="F")
    port_lib().orc_kronsumv_f64(ctypes.c_int(V.ndim), _i64(V.shape), _ptr(V), _ptrs(As), _ptr(W))
    return W


def port_permute(T: np.ndarray, p) -> np.ndarray:
    cplx = np.iscomplexobj(T)
    T = _f(T, cplx)
    out = [T.shape[k - 1] for k in p]
    S = np.empty(out, dtype=T.dtype, order="F")
    port_lib().orc_permute(ctypes.c_int(2 if cplx else 1), ctypes.c_int(T.ndim), _i64(T.shape),
                           _i64(p), _ptr(T), _ptr(S))
    return S


def port_advection_diffusion(n: int, adv: float = 0.5) -> np.ndarray:
    A = np.empty((n, n), order="F")
    port_lib().orc_advection_diffusion(ctypes.c_int64(n), ctypes.c_double(adv), _ptr(A))
    return A


# ------------------------------------------------------ ref (the reference)

_VARIANT = {"tucker": 0, "cttucker": 1, "sequential": 2, "rvalue": 3, "kron": 4, "kronsumv": 5}


def ref_tucker(T: np.ndarray, Ls, variant: str = "tucker") -> np.ndarray:
    """ops::tucker and friends from the reference library (tucker.hpp:129-232)."""
    lib = ref_lib()
    cplx = np.iscomplexobj(T) or any(np.iscomplexobj(L) for L in Ls)
    promote = cplx and not np.iscomplexobj(T)
    Ls = [_f(L, cplx) for L in Ls]
    d = T.ndim
    adj = variant == "cttucker"
    n = [L.shape[1] if adj else L.shape[0] for L in Ls]
    if variant == "kronsumv":
        n = list(T.shape)
    if promote and variant in ("tucker", "cttucker"):
        Tr = _f(T, False)
        S = np.empty(n, dtype=np.complex128, order="F")
        _check(lib.ref_tucker_promote(ctypes.c_int(d), _i64(Tr.shape), _i64([L.shape[0] for L in Ls]),
                                      _i64([L.shape[1] for L in Ls]), _ptr(Tr), _ptrs(Ls), _ptr(S),
                                      ctypes.c_int(int(adj))))
        return S
    T = _f(T, cplx)
    S = np.empty(max(1, int(np.prod(n))) if n else 1, dtype=T.dtype)
    out_ext = (ctypes.c_int64 * d)()
    fn = lib.ref_tucker_c128 if cplx else lib.ref_tucker_f64
    _check(fn(ctypes.c_int(d), _i64(T.shape), _i64([L.shape[0] for L in Ls]),
              _i64([L.shape[1] for L in Ls]), _ptr(T), _ptrs(Ls), _ptr(S), out_ext,
              ctypes.c_int(_VARIANT[variant])))
    return S.reshape(list(out_ext), order="F")


def ref_mode_product(T: np.ndarray, L: np.ndarray, mu: int, loops: bool = False) -> np.ndarray:
    """core::mode_product (mode_product.hpp:64-77) or, with loops=True,
    reference::mode_product_loops (reference.hpp:62-80)."""
    lib = ref_lib()
    cplx = np.iscomplexobj(T) or np.iscomplexobj(L)
    T = _f(T, cplx)
    L = _f(L, cplx)
    out = list(T.shape)
    if 1 <= mu <= T.ndim:
        out[mu - 1] = L.shape[0]
    S = np.empty(int(np.prod(out)), dtype=T.dtype)
    fn = lib.ref_mode_product_c128 if cplx else lib.ref_mode_product_f64
    _check(fn(ctypes.c_int(T.ndim), _i64(T.shape), ctypes.c_int(mu), ctypes.c_int64(L.shape[0]),
              ctypes.c_int64(L.shape[1]), _ptr(T), _ptr(L), _ptr(S), ctypes.c_int(int(loops))))
    return S.reshape(out, order="F")


def ref_itucker(T: np.ndarray, Ps) -> np.ndarray:
    """ops::itucker with ops::FactorizedStack<T> (tucker.hpp:34-51, 187-204)."""
    lib = ref_lib()
    cplx = np.iscomplexobj(T) or any(np.iscomplexobj(P) for P in Ps)
    T = _f(T, cplx)
    Ps = [_f(P, cplx) for P in Ps]
    S = np.empty(T.shape, dtype=T.dtype, order="F")
    fn = lib.ref_itucker_c128 if cplx else lib.ref_itucker_f64
    _check(fn(ctypes.c_int(T.ndim), _i64(T.shape), _ptr(T), _ptrs(Ps), _ptr(S)))
    return S


def ref_lu_factor(P: np.ndarray):
    """la::lu_factor (lu.hpp:23-47): (lu, piv)."""
    lib = ref_lib()
    cplx = np.iscomplexobj(P)
    P = _f(P, cplx)
    n = P.shape[0]
    lu = np.empty(P.shape, dtype=P.dtype, order="F")
    piv = np.empty(n, dtype=np.int64)
    fn = lib.ref_lu_factor_c128 if cplx else lib.ref_lu_factor_f64
    _check(fn(ctypes.c_int64(n), _ptr(P), _ptr(lu), piv.ctypes.data_as(I64P)))
    return lu, piv


def ref_symtridiag_eig(diag: np.ndarray, offdiag: np.ndarray):
    """la::symtridiag_eig, EigMode::FullVectors (src/tridiag.cpp:12-90)."""
    lib = ref_lib()
    d = np.ascontiguousarray(diag, dtype=np.float64)
    e = np.ascontiguousarray(offdiag, dtype=np.float64)
    m = d.shape[0]
    w = np.empty(m)
    V = np.empty((m, m), order="F")
    ep = e if m > 1 else np.zeros(1)
    _check(lib.ref_symtridiag_eig_f64(ctypes.c_int64(m), _ptr(d), _ptr(ep), _ptr(w), _ptr(V)))
    return w, V


def ref_imex_direct(u0: np.ndarray, As, tau: float, steps: int = 1) -> np.ndarray:
    """apps::imex_evolve with ImexBackend::Direct and no nonlinearity
    (src/imex.cpp:88-200): `steps` DirectSolver solves (:53-86) with
    M_mu = (1/d) I - tau A_mu."""
    lib = ref_lib()
    u0 = _f(u0, False)
    As = [_f(A, False) for A in As]
    u = np.empty(u0.shape, order="F")
    _check(lib.ref_imex_direct_f64(ctypes.c_int(u0.ndim), _i64(u0.shape), _ptrs(As), _ptr(u0),
                                   ctypes.c_double(tau), ctypes.c_int(steps), _ptr(u)))
    return u


def ref_expm(A: np.ndarray) -> np.ndarray:
    lib = ref_lib()
    A = _f(A, False)
    E = np.empty(A.shape, order="F")
    _check(lib.ref_expm_f64(ctypes.c_int64(A.shape[0]), _ptr(A), _ptr(E)))
    return E


def ref_laplacian(n: int) -> np.ndarray:
    lib = ref_lib()
    A = np.empty((n, n), order="F")
    _check(lib.ref_laplacian_f64(ctypes.c_int64(n), _ptr(A)))
    return A


def ref_time_tucker(T: np.ndarray, Ls, steps: int = 1, reps: int = 3):
    """Median wall time of `steps` chained ops::tucker calls (the reference's
    time_median protocol, tools/mumode_cli.cpp:79-90). Returns (median_s,
    final tensor)."""
    lib = ref_lib()
    cplx = np.iscomplexobj(T) or any(np.iscomplexobj(L) for L in Ls)
    T = _f(T, cplx)
    Ls = [_f(L, cplx) for L in Ls]
    n = [L.shape[0] for L in Ls]
    S = np.empty(n, dtype=T.dtype, order="F")
    med = ctypes.c_double()
    if cplx:
        if steps != 1:
            raise ValueError("complex timing supports steps=1")
        _check(lib.ref_time_tucker_c128(ctypes.c_int(T.ndim), _i64(T.shape), _i64(n),
                                        _i64([L.shape[1] for L in Ls]), _ptr(T), _ptrs(Ls),
                                        ctypes.c_int(reps), _ptr(S), ctypes.byref(med)))
    else:
        _check(lib.ref_time_tucker_f64(ctypes.c_int(T.ndim), _i64(T.shape), _i64(n),
                                       _i64([L.shape[1] for L in Ls]), _ptr(T), _ptrs(Ls),
                                       ctypes.c_int(steps), ctypes.c_int(reps), _ptr(S),
                                       ctypes.byref(med), None))
    return med.value, S


def ref_bench_tucker(seed: int, m, n, warmup: int, reps: int):
    """bench.py's reference arm in one call into the reference library: inputs
    drawn there with the reference's generator, `warmup` untimed then `reps`
    individually timed ops::tucker applications. Returns (per-rep seconds,
    checksum of the last result)."""
    lib = ref_lib()
    times = np.zeros(max(reps, 1))
    chk = ctypes.c_double()
    _check(lib.ref_bench_tucker_f64(ctypes.c_uint64(seed), ctypes.c_int(len(m)), _i64(m), _i64(n),
                                    ctypes.c_int(warmup), ctypes.c_int(reps), _ptr(times), ctypes.byref(chk)))
    return times[:reps], chk.value


def ref_blas_kernel_name() -> str:
    return ref_lib().ref_blas_kernel_name().decode()


# ------------------------------------------------------------ comparisons

def rel_max(a: np.ndarray, b: np.ndarray) -> float:
    """max|a-b| / max|b| (the reference tests' rel_err, test_tucker_ops.cpp:34-37)."""
    scale = max(float(np.max(np.abs(b))) if b.size else 0.0, 1e-300)
    return float(np.max(np.abs(a - b))) / scale if a.size else 0.0


def rel_fro(a: np.ndarray, b: np.ndarray) -> float:
    """||a-b||_F / ||b||_F (the north-star parity metric, gate 1e-12)."""
    nb = float(np.linalg.norm(b.ravel()))
    return float(np.linalg.norm((a - b).ravel())) / max(nb, 1e-300)
