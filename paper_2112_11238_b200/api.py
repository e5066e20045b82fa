"""Reference-shaped Python API over the B200 mu-mode engine.

Names, argument meaning and error behaviour mirror the reference library's
hot-path operators (``/root/reference/proj/include/mumode``):

=====================  ==================================================
this module            reference
=====================  ==================================================
``mode_product``       ``core::mode_product`` (mode_product.hpp:64-83)
``tucker``             ``ops::tucker`` (tucker.hpp:129-144)
``cttucker``           ``ops::cttucker`` (tucker.hpp:149-155)
``tucker_sequential``  ``ops::tucker_sequential`` (tucker.hpp:159-167)
``kronsumv``           ``ops::kronsumv`` (tucker.hpp:209-232)
``expint``             repeated ``apps::linear_evolution_exact`` step
                       (src/evolution.cpp:70-82) with precomputed factors
``expm``               ``la::expm`` role (src/expm.cpp:97-151), host
``FactorizedStack``    ``ops::FactorizedStack<T>`` (tucker.hpp:34-51)
``itucker``            ``ops::itucker`` (tucker.hpp:187-204)
``KronSumSolver``      IMEX ``DirectSolver`` (src/imex.cpp:53-86)
``SizeError`` ...      ``mumode::SizeError`` ... (errors.hpp:8-26)
=====================  ==================================================

Data model: a tensor is column-major (first index fastest,
shape.hpp:68-77). Two kinds of argument are accepted:

* ``torch.Tensor`` on a CUDA device (float64 / complex128) whose strides are
  column-major -- the device-resident path; results are new column-major CUDA
  tensors and the call is ordered on torch's current stream;
* ``numpy.ndarray`` -- the host drop-in path: the C-ABI copies host->device,
  computes, and copies back (what a reference user switching libraries gets).

Every computation runs in the CUDA kernels of ``libmumode_b200.so``; there is
no CPU fallback.
"""
from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np

from . import _lib

try:  # torch is plumbing for device memory and streams
    import torch
except ImportError:  # pragma: no cover
    torch = None


# ------------------------------------------------------------------ errors
class MumodeError(Exception):
    pass


class SizeError(MumodeError, ValueError):
    """Shape or dimension mismatch (errors.hpp:8-11)."""


class ArgumentError(MumodeError, ValueError):
    """Invalid argument value, e.g. a bad mode index (errors.hpp:13-16)."""


class ContractError(MumodeError):
    """A caller-supplied operator violated its contract (errors.hpp:23-26)."""


class NumericalError(MumodeError, ArithmeticError):
    """Numerical failure (errors.hpp:18-21)."""


class CudaError(MumodeError, RuntimeError):
    pass


_CODES = {1: SizeError, 2: ArgumentError, 3: CudaError, 4: CudaError, 5: CudaError,
          6: ContractError, 7: NumericalError}


def _check(rc: int) -> None:
    if rc != 0:
        msg = _lib.lib().mumode_last_error().decode()
        raise _CODES.get(rc, MumodeError)(msg)


# ------------------------------------------------------------------ handles
class Handle:
    """Owns a C-ABI handle (workspace, TMA descriptors, graphs) for one GPU."""

    def __init__(self, device: int = 0):
        self.device = device
        h = ctypes.c_void_p()
        _check(_lib.lib().mumode_handle_create(ctypes.byref(h), int(device)))
        self.h = h

    def bind_stream(self, stream_ptr: int | None) -> None:
        _check(_lib.lib().mumode_set_stream(self.h, ctypes.c_void_p(stream_ptr or 0)))

    def bind_torch_stream(self) -> None:
        s = torch.cuda.current_stream(self.device)
        self.bind_stream(s.cuda_stream)

    @property
    def launches(self) -> int:
        return int(_lib.lib().mumode_launch_count(self.h))

    def set_kernel_policy(self, policy: int) -> None:
        """Kernel path selection for tests / benchmarks (include/mumode_gpu.h):
        0 auto, 1 SIMT kernel, 2 TMA/DMMA where legal, 3..6 one TMA tile
        config forced, 7 auto incl. fused pairs, 8 LDG-staged DMMA, 9 / 10 tail
        pass forced / disabled, 11 whole chains as one persistent launch, 12
        fused passes without warp specialisation, 13 no skinny small-extent
        kernel, 14 no small-extent fused pairs, 15 small-extent fused pairs
        wherever eligible."""
        _check(_lib.lib().mumode_set_kernel_policy(self.h, int(policy)))

    def close(self) -> None:
        if self.h:
            _lib.lib().mumode_handle_destroy(self.h)
            self.h = None


import threading

# One handle (workspaces, descriptor cache, graphs) per thread and device: the
# reference's operators are pure functions safe for concurrent callers
# (SPEC.md:134-135), so concurrent threads must never share a workspace.
_tls = threading.local()


def get_handle(device: int | None = None) -> Handle:
    if device is None:
        device = torch.cuda.current_device() if torch is not None and torch.cuda.is_available() else 0
    handles = getattr(_tls, "handles", None)
    if handles is None:
        handles = _tls.handles = {}
    if device not in handles:
        handles[device] = Handle(device)
    return handles[device]


# ------------------------------------------------------------------ layout helpers
def colmajor_strides(shape: Sequence[int]) -> tuple[int, ...]:
    s, out = 1, []
    for e in shape:
        out.append(s)
        s *= int(e)
    return tuple(out)


def is_colmajor(t) -> bool:
    if t.dim() == 0:
        return True
    return all(st == cs or sh == 1 for st, cs, sh in zip(t.stride(), colmajor_strides(t.shape), t.shape))


def colmajor_empty(shape: Sequence[int], dtype=None, device=None):
    """Uninitialised column-major CUDA tensor with the given extents."""
    shape = [int(e) for e in shape]
    base = torch.empty(list(reversed(shape)), dtype=dtype or torch.float64, device=device)
    return base.permute(*reversed(range(len(shape))))


def to_colmajor(t):
    """Column-major copy (or the tensor itself if already column-major)."""
    if is_colmajor(t):
        return t
    out = colmajor_empty(t.shape, t.dtype, t.device)
    out.copy_(t)
    return out


def _is_torch(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor)


def _dev_ptr(t) -> int:
    return t.data_ptr()


def _np_f(a, cplx: bool) -> np.ndarray:
    return np.asfortranarray(a, dtype=np.complex128 if cplx else np.float64)


def _is_cplx(x) -> bool:
    if _is_torch(x):
        return x.is_complex()
    return np.iscomplexobj(x)


def _extents(x) -> list[int]:
    return [int(e) for e in x.shape]


def _validate_tensor(T):
    if T.ndim < 1 or any(int(e) < 1 for e in T.shape):
        raise ArgumentError("tensor order must be >= 1" if T.ndim < 1 else "tensor extents must be positive")
    if _is_torch(T):
        if not T.is_cuda:
            raise ArgumentError("torch tensors must live on a CUDA device (the engine has no CPU path)")
        if T.dtype not in (torch.float64, torch.complex128):
            raise ArgumentError("tensors must be float64 or complex128")


def _validate_matrix(L):
    if L.ndim != 2:
        raise ArgumentError("factor matrices must be 2-D")
    if int(L.shape[0]) < 1 or int(L.shape[1]) < 1:
        raise ArgumentError("matrix dimensions must be positive")


def _dev_matrix(L, cplx: bool, device):
    """Column-major CUDA copy of a factor (tiny) in the right dtype."""
    dt = torch.complex128 if cplx else torch.float64
    if not _is_torch(L):
        L = torch.from_numpy(np.ascontiguousarray(np.asarray(L)))
    L = L.to(device=device, dtype=dt)
    return to_colmajor(L)


# ------------------------------------------------------------------ operators
def mode_product(T, L, mu: int):
    """S = T x_mu L (core::mode_product, mode_product.hpp:64-83).

    L is n x m_mu; a real tensor with a complex matrix promotes to complex
    (mode_product.hpp:80-83)."""
    _validate_tensor(T)
    _validate_matrix(L)
    d = T.ndim
    if mu < 1 or mu > d:
        raise ArgumentError(f"mode index {mu} out of range 1..{d}")
    if int(L.shape[1]) != int(T.shape[mu - 1]):
        raise SizeError(f"mode_product: matrix columns ({int(L.shape[1])}) do not match extent of mode {mu}")
    cplx = _is_cplx(T) or _is_cplx(L)
    m = _extents(T)
    n_mu = int(L.shape[0])
    out_ext = list(m)
    out_ext[mu - 1] = n_mu
    lib = _lib.lib()
    if _is_torch(T):
        h = get_handle(T.device.index)
        h.bind_torch_stream()
        Td = to_colmajor(T.to(torch.complex128) if cplx and not T.is_complex() else T)
        Ld = _dev_matrix(L, cplx, T.device)
        S = colmajor_empty(out_ext, Td.dtype, T.device)
        fn = lib.mumode_mode_product_c128 if cplx else lib.mumode_mode_product_f64
        _check(fn(h.h, d, _lib.i64_array(m), mu, n_mu, _dev_ptr(Td), _dev_ptr(Ld), _dev_ptr(S)))
        return S
    h = get_handle()
    Tn = _np_f(T, cplx)
    Ln = _np_f(L, cplx)
    S = np.empty(out_ext, dtype=Tn.dtype, order="F")
    fn = lib.mumode_host_mode_product_c128 if cplx else lib.mumode_host_mode_product_f64
    _check(fn(h.h, d, _lib.i64_array(m), mu, n_mu, Tn.ctypes.data, Ln.ctypes.data, S.ctypes.data))
    return S


def _check_stack(T, Ls, adjoint: bool, who: str = "tucker"):
    d = T.ndim
    if len(Ls) != d:
        raise SizeError(f"{who}: stack holds {len(Ls)} matrices for an order-{d} tensor")
    for mu in range(1, d + 1):
        L = Ls[mu - 1]
        _validate_matrix(L)
        need = int(L.shape[0]) if adjoint else int(L.shape[1])
        if need != int(T.shape[mu - 1]):
            raise SizeError(f"{who}: matrix for mode {mu} expects extent {need}, tensor has {int(T.shape[mu - 1])}")


def _tucker_impl(T, Ls, adjoint: bool):
    _validate_tensor(T)
    Ls = list(Ls)
    _check_stack(T, Ls, adjoint)
    d = T.ndim
    cplx_L = any(_is_cplx(L) for L in Ls)
    cplx = _is_cplx(T) or cplx_L
    promote = cplx_L and not _is_cplx(T)
    m = _extents(T)
    n = [int(L.shape[1]) if adjoint else int(L.shape[0]) for L in Ls]
    lib = _lib.lib()
    if _is_torch(T):
        h = get_handle(T.device.index)
        h.bind_torch_stream()
        Td = to_colmajor(T)
        if cplx and not promote and not Td.is_complex():
            Td = Td.to(torch.complex128)
        Lds = [_dev_matrix(L, cplx, T.device) for L in Ls]
        S = colmajor_empty(n, torch.complex128 if cplx else torch.float64, T.device)
        if promote:
            fn = lib.mumode_tucker_promote
        else:
            fn = lib.mumode_tucker_c128 if cplx else lib.mumode_tucker_f64
        _check(fn(h.h, d, _lib.i64_array(m), _lib.i64_array(n), _dev_ptr(Td),
                  _lib.ptr_array([_dev_ptr(L) for L in Lds]), _dev_ptr(S), int(adjoint)))
        return S
    h = get_handle()
    Tn = _np_f(T, cplx and not promote)
    Lns = [_np_f(L, cplx) for L in Ls]
    S = np.empty(n, dtype=np.complex128 if cplx else np.float64, order="F")
    if promote:
        fn = lib.mumode_host_tucker_promote
    else:
        fn = lib.mumode_host_tucker_c128 if cplx else lib.mumode_host_tucker_f64
    _check(fn(h.h, d, _lib.i64_array(m), _lib.i64_array(n), Tn.ctypes.data,
              _lib.ptr_array([L.ctypes.data for L in Lns]), S.ctypes.data, int(adjoint)))
    return S


def tucker(T, Ls):
    """S = T x_1 L_1 x_2 ... x_d L_d (ops::tucker, tucker.hpp:129-144).
    L_mu is n_mu x m_mu. Real T with complex L promotes to complex."""
    return _tucker_impl(T, Ls, adjoint=False)


def cttucker(T, Psis):
    """S = T x_1 Psi_1^H ... x_d Psi_d^H (ops::cttucker, tucker.hpp:149-155);
    Psi_mu is m_mu x n_mu and no Psi^H is formed by the caller."""
    return _tucker_impl(T, Psis, adjoint=True)


def tucker_sequential(T, Ls):
    """Unfused chain of standalone mode products (tucker.hpp:159-167)."""
    _validate_tensor(T)
    if len(Ls) != T.ndim:
        raise SizeError("tucker_sequential: stack length")
    cur = mode_product(T, Ls[0], 1)
    for mu in range(2, T.ndim + 1):
        cur = mode_product(cur, Ls[mu - 1], mu)
    return cur


def kronsumv(V, As):
    """W = sum_mu V x_mu A_mu (ops::kronsumv, tucker.hpp:209-232), real or
    complex (mixed operands promote to complex)."""
    _validate_tensor(V)
    d = V.ndim
    As = list(As)
    if len(As) != d:
        raise SizeError("kronsumv: stack length does not match tensor order")
    for mu in range(1, d + 1):
        A = As[mu - 1]
        _validate_matrix(A)
        if int(A.shape[0]) != int(A.shape[1]):
            raise SizeError(f"kronsumv: matrix for mode {mu} is not square")
        if int(A.shape[1]) != int(V.shape[mu - 1]):
            raise SizeError(f"kronsumv: matrix size does not match extent of mode {mu}")
    cplx = _is_cplx(V) or any(_is_cplx(A) for A in As)
    m = _extents(V)
    lib = _lib.lib()
    if _is_torch(V):
        h = get_handle(V.device.index)
        h.bind_torch_stream()
        Vd = to_colmajor(V.to(torch.complex128) if cplx and not V.is_complex() else V)
        Ads = [_dev_matrix(A, cplx, V.device) for A in As]
        W = colmajor_empty(m, Vd.dtype, V.device)
        fn = lib.mumode_kronsumv_c128 if cplx else lib.mumode_kronsumv_f64
        _check(fn(h.h, d, _lib.i64_array(m), _dev_ptr(Vd), _lib.ptr_array([_dev_ptr(A) for A in Ads]), _dev_ptr(W)))
        return W
    h = get_handle()
    Vn = _np_f(V, cplx)
    Ans = [_np_f(A, cplx) for A in As]
    W = np.empty(m, dtype=Vn.dtype, order="F")
    fn = lib.mumode_host_kronsumv_c128 if cplx else lib.mumode_host_kronsumv_f64
    _check(fn(h.h, d, _lib.i64_array(m), Vn.ctypes.data, _lib.ptr_array([A.ctypes.data for A in Ans]),
              W.ctypes.data))
    return W


def expint(u0, Es, steps: int, out=None):
    """Exponential-integrator march: u <- tucker(u; E_1..E_d), `steps` times
    (the Tucker step of apps::linear_evolution_exact, src/evolution.cpp:70-82,
    with E_mu = expm(tau A_mu) precomputed). Replayed as one CUDA graph."""
    _validate_tensor(u0)
    d = u0.ndim
    Es = list(Es)
    _check_stack(u0, Es, False, who="expint")
    for mu, E in enumerate(Es, 1):
        if int(E.shape[0]) != int(E.shape[1]):
            raise SizeError(f"expint: matrix for mode {mu} is not square")
    m = _extents(u0)
    lib = _lib.lib()
    if _is_torch(u0):
        h = get_handle(u0.device.index)
        h.bind_torch_stream()
        ud = to_colmajor(u0)
        Eds = [_dev_matrix(E, False, u0.device) for E in Es]
        if out is None:
            out = colmajor_empty(m, torch.float64, u0.device)
        _check(lib.mumode_expint_f64(h.h, d, _lib.i64_array(m),
                                     _lib.ptr_array([_dev_ptr(E) for E in Eds]), _dev_ptr(ud),
                                     _dev_ptr(out), int(steps)))
        return out
    h = get_handle()
    un = _np_f(u0, False)
    Ens = [_np_f(E, False) for E in Es]
    res = np.empty(m, order="F")
    _check(lib.mumode_host_expint_f64(h.h, d, _lib.i64_array(m),
                                      _lib.ptr_array([E.ctypes.data for E in Ens]), un.ctypes.data,
                                      res.ctypes.data, int(steps)))
    return res


def matricize(T, mu: int):
    """mu-matricization (core::matricize, matricize.hpp:22-31): the
    m_mu x (prod of the other extents) matrix of mu-fibres, columns ordered by
    the remaining indices with the earliest fastest. Host-side helper for
    user callbacks (numpy in, numpy out)."""
    T = np.asarray(T.cpu() if _is_torch(T) else T)
    d = T.ndim
    if mu < 1 or mu > d:
        raise ArgumentError(f"mode index {mu} out of range 1..{d}")
    order = [mu - 1] + [k for k in range(d) if k != mu - 1]
    return np.asfortranarray(np.transpose(T, order).reshape((T.shape[mu - 1], -1), order="F"))


def dematricize(M, mu: int, shape):
    """Inverse of matricize (matricize.hpp:35-56); the output's extent mu is
    M's row count."""
    M = np.asarray(M)
    shape = [int(e) for e in shape]
    d = len(shape)
    if mu < 1 or mu > d:
        raise ArgumentError(f"mode index {mu} out of range 1..{d}")
    rest = [shape[k] for k in range(d) if k != mu - 1]
    if M.shape[1] != int(np.prod(rest)):
        raise SizeError("dematricize: column count does not match remaining extents")
    fronted = M.reshape([M.shape[0]] + rest, order="F")
    inv = np.argsort([mu - 1] + [k for k in range(d) if k != mu - 1])
    return np.asfortranarray(np.transpose(fronted, inv))


def mode_action(T, op, mu: int):
    """mu-mode action (core::mode_action, mode_product.hpp:88-100): a columnwise
    host operator on the mu-matricization."""
    X = matricize(T, mu)
    Y = np.asarray(op(X))
    if Y.ndim != 2 or Y.shape[1] != X.shape[1]:
        raise ContractError(f"mode_action: operator changed the column count on mode {mu}")
    return dematricize(Y, mu, np.asarray(T.cpu() if _is_torch(T) else T).shape)


def tuckerfun(T, ops):
    """Operator-action Tucker (ops::tuckerfun, tucker.hpp:169-185): ``ops`` is a
    list of (out_rows, callable) per mode, applied in mode order. Host
    callbacks, so this runs on the host (not the accelerated path)."""
    T = np.asarray(T.cpu() if _is_torch(T) else T)
    if len(ops) != T.ndim:
        raise SizeError("tuckerfun: stack length does not match tensor order")
    cur = T
    for mu, (out_rows, fn) in enumerate(ops, start=1):
        cur = mode_action(cur, fn, mu)
        if cur.shape[mu - 1] != out_rows:
            raise ContractError(f"tuckerfun: operator on mode {mu} produced {cur.shape[mu - 1]} rows, "
                                f"declared {out_rows}")
    return cur


class FactorizedStack:
    """Per-mode LU factorizations of square P_1..P_d for the inverse Tucker
    operator (ops::FactorizedStack<T>, tucker.hpp:34-51). Factorizes at
    construction exactly as la::lu_factor (lu.hpp:23-47; host,
    mumode_lu_factor_*), raising NumericalError on a singular pivot (lu.hpp:33)
    and SizeError for a non-square factor. The stack is complex if any P_mu
    is. ``factor(mu)`` returns (lu, piv) like the reference's ``factor``."""

    def __init__(self, Ps):
        Ps = [np.asarray(P.cpu() if _is_torch(P) else P) for P in Ps]
        self.cplx = any(np.iscomplexobj(P) for P in Ps)
        self.lu, self.piv = [], []
        fn = _lib.lib().mumode_lu_factor_c128 if self.cplx else _lib.lib().mumode_lu_factor_f64
        for P in Ps:
            Pn = _np_f(P, self.cplx)
            if Pn.ndim != 2 or Pn.shape[0] != Pn.shape[1]:
                raise SizeError("lu_factor: matrix must be square")
            lu = np.empty(Pn.shape, dtype=Pn.dtype, order="F")
            piv = np.empty(Pn.shape[0], dtype=np.int64)
            _check(fn(int(Pn.shape[0]), Pn.ctypes.data, lu.ctypes.data, piv.ctypes.data))
            self.lu.append(lu)
            self.piv.append(piv)
        self._dev = {}

    def size(self) -> int:
        return len(self.lu)

    def factor(self, mu: int):
        return self.lu[mu - 1], self.piv[mu - 1]

    def _device(self, device, cplx: bool):
        key = (str(device), cplx)
        if key not in self._dev:
            dt = torch.complex128 if cplx else torch.float64
            self._dev[key] = ([torch.from_numpy(lu).to(device=device, dtype=dt) for lu in self.lu],
                              [torch.from_numpy(p).to(device) for p in self.piv])
        return self._dev[key]


def itucker(T, F: FactorizedStack):
    """S = T x_1 P_1^-1 ... x_d P_d^-1 (ops::itucker, tucker.hpp:187-204):
    per-mode triangular solves with the stored factors on the GPU (no inverse
    is formed). A real tensor with a complex stack promotes to complex."""
    _validate_tensor(T)
    if F.size() != T.ndim:
        raise SizeError("itucker: stack length does not match tensor order")
    for mu, lu in enumerate(F.lu, 1):
        if lu.shape[0] != int(T.shape[mu - 1]):
            raise SizeError(f"itucker: factor size does not match extent of mode {mu}")
    cplx = F.cplx or _is_cplx(T)
    m = _extents(T)
    lib = _lib.lib()
    if _is_torch(T):
        h = get_handle(T.device.index)
        h.bind_torch_stream()
        Td = to_colmajor(T.to(torch.complex128) if cplx and not T.is_complex() else T)
        lus, pivs = F._device(T.device, cplx)
        S = colmajor_empty(m, Td.dtype, T.device)
        fn = lib.mumode_itucker_c128 if cplx else lib.mumode_itucker_f64
        _check(fn(h.h, T.ndim, _lib.i64_array(m), _dev_ptr(Td), _lib.ptr_array([_dev_ptr(x) for x in lus]),
                  _lib.ptr_array([_dev_ptr(p) for p in pivs]), _dev_ptr(S)))
        return S
    h = get_handle()
    Tn = _np_f(T, cplx)
    lus = [_np_f(lu, cplx) for lu in F.lu]
    S = np.empty(m, dtype=Tn.dtype, order="F")
    fn = lib.mumode_host_itucker_c128 if cplx else lib.mumode_host_itucker_f64
    _check(fn(h.h, T.ndim, _lib.i64_array(m), Tn.ctypes.data, _lib.ptr_array([x.ctypes.data for x in lus]),
              _lib.ptr_array([p.ctypes.data for p in F.piv]), S.ctypes.data))
    return S


def extract_tridiag(M):
    """Symmetric tridiagonal part (diag, offdiag) of a factor M -- the IMEX
    direct backend's extract_tridiag (src/imex.cpp:28-48), with its
    ArgumentError for entries off the three diagonals or an asymmetric pair."""
    Mn = _np_f(np.asarray(M.cpu() if _is_torch(M) else M), False)
    if Mn.ndim != 2 or Mn.shape[0] != Mn.shape[1]:
        raise SizeError("extract_tridiag: matrix must be square")
    n = int(Mn.shape[0])
    diag = np.empty(n)
    off = np.empty(max(n - 1, 1))
    _check(_lib.lib().mumode_extract_tridiag_f64(n, Mn.ctypes.data, diag.ctypes.data, off.ctypes.data))
    return diag, off[:n - 1]


def symtridiag_eig(diag, offdiag):
    """Ascending eigenvalues and eigenvector columns of a symmetric
    tridiagonal matrix (la::symtridiag_eig with EigMode::FullVectors,
    src/tridiag.cpp:12-90: implicit-shift QL, bitwise the reference's)."""
    d = np.ascontiguousarray(diag, dtype=np.float64)
    e = np.ascontiguousarray(offdiag, dtype=np.float64)
    m = int(d.shape[0])
    if m < 1:
        raise ArgumentError("symtridiag_eig: empty matrix")
    if int(e.shape[0]) != m - 1:
        raise ArgumentError("symtridiag_eig: offdiag must have one entry fewer than diag")
    w = np.empty(m)
    V = np.empty((m, m), order="F")
    ep = e if m > 1 else np.zeros(1)
    _check(_lib.lib().mumode_symtridiag_eig_f64(m, d.ctypes.data, ep.ctypes.data, w.ctypes.data, V.ctypes.data))
    return w, V


class KronSumSolver:
    """Direct solver for (sum_mu I x ... x M_mu x ... x I) x = b -- the IMEX
    direct backend (DirectSolver, src/imex.cpp:53-86). Built from the factors
    M_mu exactly as the reference builds it: extract_tridiag (ArgumentError
    unless M_mu is symmetric tridiagonal), symtridiag_eig (implicit-shift QL)
    and Q_mu^T; or from given eigenpairs (Qs, evals). Each solve is two Tucker
    applications around a pointwise division by the eigenvalue Kronecker sum,
    on the GPU (mumode_kronsum_solve_f64)."""

    def __init__(self, Ms=None, Qs=None, evals=None, device=None):
        if Ms is not None:
            Qs, evals = [], []
            for M in Ms:
                w, V = symtridiag_eig(*extract_tridiag(M))
                Qs.append(V)
                evals.append(w)
        if Qs is None or evals is None or len(Qs) != len(evals):
            raise ArgumentError("kronsum_solve: need the factors Ms, or eigenvectors and eigenvalues per mode")
        self.evals = [np.ascontiguousarray(np.asarray(e, dtype=np.float64)) for e in evals]
        self.Q = [np.asfortranarray(np.asarray(Q, dtype=np.float64)) for Q in Qs]
        for mu, (Q, e) in enumerate(zip(self.Q, self.evals), 1):
            if Q.ndim != 2 or Q.shape[0] != Q.shape[1] or e.shape != (Q.shape[0],):
                raise SizeError(f"kronsum_solve: eigenpairs of mode {mu} do not match")
        self.Qt = [np.asfortranarray(Q.T) for Q in self.Q]
        self._dev = {}

    def _device_mats(self, device):
        key = str(device)
        if key not in self._dev:
            self._dev[key] = ([torch.from_numpy(Q).to(device) for Q in self.Q],
                              [torch.from_numpy(Q).to(device) for Q in self.Qt])
        return self._dev[key]

    def solve(self, b):
        _validate_tensor(b)
        d = b.ndim
        if len(self.Q) != d:
            raise SizeError("kronsum_solve: stack length does not match tensor order")
        for mu in range(1, d + 1):
            if self.Q[mu - 1].shape != (int(b.shape[mu - 1]),) * 2:
                raise SizeError(f"kronsum_solve: factor size does not match extent of mode {mu}")
        m = _extents(b)
        host_in = not _is_torch(b)
        bd = torch.from_numpy(_np_f(b, False)).cuda() if host_in else to_colmajor(b)
        h = get_handle(bd.device.index)
        h.bind_torch_stream()
        Qd, Qtd = self._device_mats(bd.device)
        x = colmajor_empty(m, torch.float64, bd.device)
        ev_ptrs = _lib.ptr_array([e.ctypes.data for e in self.evals])
        _check(_lib.lib().mumode_kronsum_solve_f64(
            h.h, d, _lib.i64_array(m), _lib.ptr_array([Q.data_ptr() for Q in Qd]),
            _lib.ptr_array([Q.data_ptr() for Q in Qtd]), ev_ptrs, bd.data_ptr(), x.data_ptr()))
        return x.cpu().numpy() if host_in else x


def expm(A) -> np.ndarray:
    """Matrix exponential on the host (scaling and squaring, Pade 13)."""
    An = _np_f(np.asarray(A), False)
    if An.ndim != 2 or An.shape[0] != An.shape[1]:
        raise SizeError("expm: matrix is not square")
    E = np.empty(An.shape, order="F")
    _check(_lib.lib().mumode_expm_f64(int(An.shape[0]), An.ctypes.data, E.ctypes.data))
    return E


# ------------------------------------------------------------------ inputs
class Rng:
    """The reference's input generator: std::mt19937_64(seed) with a fresh
    std::normal_distribution<double> per filled object, column-major fill,
    complex entries drawing re then im (tools/mumode_cli.cpp:92-121)."""

    def __init__(self, seed: int):
        r = ctypes.c_void_p()
        _check(_lib.lib().mumode_rng_create(ctypes.byref(r), ctypes.c_uint64(seed)))
        self.r = r

    def __del__(self):
        try:
            if getattr(self, "r", None):
                _lib.lib().mumode_rng_destroy(self.r)
                self.r = None
        except Exception:  # interpreter shutdown
            pass

    def normal(self, shape, complex_: bool = False, out: np.ndarray | None = None) -> np.ndarray:
        shape = [int(e) for e in shape]
        if out is None:
            out = np.empty(shape, dtype=np.complex128 if complex_ else np.float64, order="F")
        n = int(np.prod(shape)) if shape else 1
        _check(_lib.lib().mumode_rng_normal(self.r, out.ctypes.data, n, int(complex_)))
        return out

    def u64(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        _check(_lib.lib().mumode_rng_u64(self.r, out.ctypes.data, n))
        return out


def launch_count(device: int = 0) -> int:
    return get_handle(device).launches
