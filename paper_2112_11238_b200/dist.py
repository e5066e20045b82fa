"""Slab-partitioned Tucker operator across GPUs.

A tensor too large for one GPU (or a Tucker application spread for speed) is
partitioned over its LAST mode: rank r holds the slab T[..., c_r] with the
full extents of modes 1..d-1. One application S = T x_1 L_1 ... x_d L_d is

1. local:     Y_r = T_r x_1 L_1 ... x_{d-1} L_{d-1}     (no communication;
              mumode_tucker_range_f64, the TMA/DMMA kernels)
2. exchange:  view Y_r as a column-major (A x c_r) matrix, A = n_1...n_{d-1};
              split the rows A into P blocks A_q and send block q to rank q
              (mumode_slab_pack_f64 + one all-to-all over NCCL / NVLink).
              Rank r receives, in rank order, the blocks (A_r x c_s) -- which,
              laid side by side, ARE the column-major (A_r x m_d) matrix: the
              last mode is now local.
3. local:     S_r = Y[A_r, :] x_2 L_d  ->  (A_r x n_d), rows A_r of the
              flattened result (mumode_mode_product_f64 on the 2-D view).

The output stays row-partitioned over the flattened leading modes;
``gather_rows`` reassembles it (used by the parity tests). The exchange moves
(P-1)/P of each slab; for C2 on 8 GPUs that is 14.7 MB per rank.

The algorithm is written once against a small backend interface so the
partition/exchange/assembly logic runs identically with the CUDA + NCCL
backend (``CudaSlabBackend``, the product) and with a CPU test backend over
gloo that lives in tests/ (there is no CPU backend in the product).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np


def even_splits(total: int, parts: int) -> list[int]:
    base, extra = divmod(int(total), int(parts))
    return [base + (1 if q < extra else 0) for q in range(parts)]


def offsets(sizes: Sequence[int]) -> list[int]:
    off = [0]
    for s in sizes:
        off.append(off[-1] + int(s))
    return off


@dataclass
class SlabPlan:
    """Partition of one Tucker application over P ranks."""

    m: tuple[int, ...]  # input extents
    n: tuple[int, ...]  # output extents
    P: int

    def __post_init__(self):
        self.m = tuple(int(e) for e in self.m)
        self.n = tuple(int(e) for e in self.n)
        if len(self.m) < 2:
            raise ValueError("slab partitioning needs an order >= 2 tensor")
        if self.m[-1] < self.P:
            raise ValueError(f"last mode extent {self.m[-1]} < {self.P} ranks")
        self.c_sizes = even_splits(self.m[-1], self.P)     # input slabs (last mode)
        self.c_off = offsets(self.c_sizes)
        self.A = int(np.prod(self.n[:-1]))                  # flattened leading extent after step 1
        self.a_sizes = even_splits(self.A, self.P)          # output row blocks
        self.a_off = offsets(self.a_sizes)

    def local_in_extents(self, r: int) -> tuple[int, ...]:
        return self.m[:-1] + (self.c_sizes[r],)

    def send_counts(self, r: int) -> list[int]:
        return [a * self.c_sizes[r] for a in self.a_sizes]

    def recv_counts(self, r: int) -> list[int]:
        return [self.a_sizes[r] * c for c in self.c_sizes]

    def out_rows(self, r: int) -> tuple[int, int]:
        return self.a_off[r], self.a_off[r + 1]

    def flops(self) -> float:
        ext, f = list(self.m), 0.0
        for mu in range(len(self.m)):
            f += 2.0 * self.n[mu] * float(np.prod(ext))
            ext[mu] = self.n[mu]
        return f

    def exchange_bytes(self, r: int, elem: int = 8) -> int:
        """Bytes rank r sends to other ranks."""
        return sum(c for q, c in enumerate(self.send_counts(r)) if q != r) * elem


def slab_tucker(plan: SlabPlan, rank: int, T_local, Ls, backend):
    """One slab-partitioned Tucker application on rank `rank`. Returns the
    (A_r x n_d) row block of the flattened result (column-major)."""
    d = len(plan.m)
    Y = backend.local_modes(T_local, plan.local_in_extents(rank), plan.n, Ls, 1, d - 1)
    send = backend.pack(Y, plan.A, plan.c_sizes[rank], plan.a_off)
    recv = backend.alltoall(send, plan.send_counts(rank), plan.recv_counts(rank))
    Z_rows = plan.a_sizes[rank]
    return backend.last_mode(recv, Z_rows, plan.m[-1], Ls[-1])


def slab_tucker_overlapped(plan: SlabPlan, rank: int, T_local, Ls, backend, chunks: int = 4):
    """Same result as ``slab_tucker`` with the exchange overlapped with the
    local contraction: each rank splits its slab's last-mode columns into
    ``chunks`` sub-slabs; sub-slab j is contracted (modes 1..d-1), packed by
    destination row block and posted as grouped send/recv while sub-slab j+1
    is contracted. Every received block (A_r x w columns) lands directly in
    its final columns of the (A_r x m_d) matrix, which are contiguous in the
    column-major layout -- no unpack. All ranks derive every other rank's
    chunking from the plan, so the posted sends and receives always match."""
    P, d = plan.P, len(plan.m)
    subs = [even_splits(c, min(chunks, c)) for c in plan.c_sizes]
    nchunks = max(len(sv) for sv in subs)
    subs = [sv + [0] * (nchunks - len(sv)) for sv in subs]
    suboffs = [offsets(sv) for sv in subs]
    A_r = plan.a_sizes[rank]
    Z = backend.empty(A_r * plan.m[-1])
    slab_rows = int(np.prod(plan.m[:-1]))
    pending = []
    for j in range(nchunks):
        w = subs[rank][j]
        if w > 0:
            Tj = backend.cols(T_local, slab_rows, suboffs[rank][j], w)
            ext = plan.m[:-1] + (w,)
            Yj = backend.local_modes(Tj, ext, plan.n, Ls, 1, d - 1)
            send = backend.pack(Yj, plan.A, w, plan.a_off)
        sends, recvs = [], []
        for q in range(P):
            if q == rank or w == 0:
                continue
            sends.append((q, backend.view(send, plan.a_off[q] * w, plan.a_off[q + 1] * w)))
        for s_ in range(P):
            ws = subs[s_][j]
            if s_ == rank or ws == 0:
                continue
            col0 = plan.c_off[s_] + suboffs[s_][j]
            recvs.append((s_, backend.view(Z, A_r * col0, A_r * (col0 + ws))))
        if w > 0:  # own block: device copy into place
            col0 = plan.c_off[rank] + suboffs[rank][j]
            backend.copy(backend.view(Z, A_r * col0, A_r * (col0 + w)),
                         backend.view(send, plan.a_off[rank] * w, plan.a_off[rank + 1] * w))
        if sends or recvs:
            pending.append(backend.post(sends, recvs))
    for handle in pending:
        backend.wait(handle)
    return backend.last_mode(Z, A_r, plan.m[-1], Ls[-1])


class CudaSlabBackend:
    """Product backend: CUDA kernels of libmumode_b200.so for the local steps,
    one NCCL all-to-all (torch.distributed) for the exchange."""

    def __init__(self, device: int, group=None):
        import torch
        import torch.distributed as dist

        from . import _lib
        from .api import get_handle

        self.torch, self.dist, self._lib = torch, dist, _lib
        self.group = group
        self.dev = torch.device("cuda", device)
        self.h = get_handle(device)
        self.lib = _lib.lib()

    def _check(self, rc):
        if rc:
            from .api import _check
            _check(rc)

    def local_modes(self, T, m, n_all, Ls, lo, hi):
        torch = self.torch
        self.h.bind_torch_stream()
        out_ext = list(m)
        for mu in range(lo, hi + 1):
            out_ext[mu - 1] = n_all[mu - 1]
        Y = torch.empty(int(np.prod(out_ext)), dtype=torch.float64, device=self.dev)
        ptrs = [L.data_ptr() for L in Ls]
        self._check(self.lib.mumode_tucker_range_f64(
            self.h.h, len(m), self._lib.i64_array(m), self._lib.i64_array(list(n_all[:-1]) + [m[-1]]),
            T.data_ptr(), self._lib.ptr_array(ptrs), Y.data_ptr(), lo, hi))
        return Y

    def pack(self, Y, A, C, a_off):
        send = self.torch.empty(A * C, dtype=self.torch.float64, device=self.dev)
        self._check(self.lib.mumode_slab_pack_f64(self.h.h, A, C, len(a_off) - 1,
                                                  self._lib.i64_array(a_off), Y.data_ptr(), send.data_ptr()))
        return send

    def alltoall(self, send, send_counts, recv_counts):
        recv = self.torch.empty(sum(recv_counts), dtype=self.torch.float64, device=self.dev)
        self.dist.all_to_all_single(recv, send, recv_counts, send_counts, group=self.group)
        return recv

    # --- overlapped variant
    def empty(self, n):
        return self.torch.empty(n, dtype=self.torch.float64, device=self.dev)

    def cols(self, T, rows_per_col, c0, w):
        # raw column-major storage (T.reshape(-1) would flatten in logical,
        # row-major order): the last-mode columns are contiguous runs
        from .api import is_colmajor
        if not is_colmajor(T):
            raise ValueError("slab tensors must be column-major")
        flat = T.as_strided((T.numel(),), (1,))
        return flat[rows_per_col * c0: rows_per_col * (c0 + w)]

    def view(self, x, lo, hi):
        return x[lo:hi]

    def copy(self, dst, src):
        dst.copy_(src)

    def post(self, sends, recvs):
        dist = self.dist
        ops = [dist.P2POp(dist.isend, t, peer, group=self.group) for peer, t in sends]
        ops += [dist.P2POp(dist.irecv, t, peer, group=self.group) for peer, t in recvs]
        return dist.batch_isend_irecv(ops)

    def wait(self, works):
        for w in works:
            w.wait()

    def last_mode(self, Z, rows, m_d, L_d):
        n_d = int(L_d.shape[0])
        S = self.torch.empty(rows * n_d, dtype=self.torch.float64, device=self.dev)
        self.h.bind_torch_stream()
        self._check(self.lib.mumode_mode_product_f64(self.h.h, 2, self._lib.i64_array([rows, m_d]), 2, n_d,
                                                     Z.data_ptr(), L_d.data_ptr(), S.data_ptr()))
        return S


# ------------------------------------------------------------------ C-ABI path
class Comm:
    """A ``mumode_comm_t``: NCCL communicator + exchange stream + buffers of the
    C-ABI slab-partitioned Tucker (``mumode_dist_tucker_{f64,c128}``)."""

    NCCL_ID_BYTES = 128

    def __init__(self, nranks: int, rank: int, unique_id: bytes | None, device: int = 0):
        import ctypes

        from . import _lib
        from .api import _check
        self.nranks, self.rank, self.device = int(nranks), int(rank), int(device)
        c = ctypes.c_void_p()
        if unique_id is None:  # single rank without NCCL
            if self.nranks != 1:
                raise ValueError("a multi-rank communicator needs an NCCL unique id")
            _check(_lib.lib().mumode_comm_wrap(ctypes.byref(c), self.device, None, 1, 0))
        else:
            buf = ctypes.create_string_buffer(bytes(unique_id), self.NCCL_ID_BYTES)
            _check(_lib.lib().mumode_comm_create(ctypes.byref(c), self.device, buf, self.nranks, self.rank))
        self.c = c

    @staticmethod
    def unique_id() -> bytes:
        import ctypes

        from . import _lib
        from .api import _check
        buf = ctypes.create_string_buffer(Comm.NCCL_ID_BYTES)
        _check(_lib.lib().mumode_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def from_torch(cls, group=None, device: int | None = None) -> "Comm":
        """Collective over a torch.distributed group: its first rank creates the
        NCCL id and broadcasts it through the group."""
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        src = dist.get_global_rank(group, 0) if group is not None else 0
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=src, group=group)
        dev = torch.cuda.current_device() if device is None else device
        return cls(world, rank, obj[0], dev)

    @classmethod
    def local(cls, nranks: int, rank: int, device: int = 0) -> "Comm":
        """A communicator without NCCL for the peer-store exchange: the caller
        moves the CUDA-IPC handles between ranks (``ipc_export`` /
        ``ipc_import``) over any transport (mumode_comm_create_local)."""
        import ctypes

        from . import _lib
        from .api import _check
        self = cls.__new__(cls)
        self.nranks, self.rank, self.device = int(nranks), int(rank), int(device)
        c = ctypes.c_void_p()
        _check(_lib.lib().mumode_comm_create_local(ctypes.byref(c), self.device, self.nranks, self.rank))
        self.c = c
        return self

    def ipc_export(self, m: Sequence[int], n: Sequence[int], cplx: bool = False) -> bytes:
        """This rank's CUDA-IPC handles (Z[0], Z[1], flags) for a shape."""
        import ctypes

        from . import _lib
        from .api import _check
        nb = _lib.lib().mumode_comm_ipc_handle_bytes()
        buf = ctypes.create_string_buffer(nb)
        _check(_lib.lib().mumode_comm_ipc_export(self.c, len(m), _lib.i64_array(m), _lib.i64_array(n), int(cplx),
                                                  buf))
        return buf.raw

    def ipc_import(self, m: Sequence[int], n: Sequence[int], handles: Sequence[bytes], cplx: bool = False) -> None:
        """Open every rank's exported handles (rank order)."""
        import ctypes

        from . import _lib
        from .api import _check
        blob = b"".join(handles)
        buf = ctypes.create_string_buffer(blob, len(blob))
        _check(_lib.lib().mumode_comm_ipc_import(self.c, len(m), _lib.i64_array(m), _lib.i64_array(n), int(cplx),
                                                  buf))

    def poll(self, timeout_ms: int = 60000, device: int | None = None) -> None:
        """Wait for this rank's queued work with NCCL failure detection
        (mumode_comm_poll): raises instead of hanging on a lost peer."""
        from . import _lib
        from .api import _check, get_handle
        h = get_handle(self.device if device is None else device)
        _check(_lib.lib().mumode_comm_poll(h.h, self.c, int(timeout_ms)))

    def set_exchange(self, mode: str) -> None:
        """'nccl' (grouped send/recv, default) or 'p2p' (the last local mode's
        epilogue stores rows straight into the owning ranks' memory)."""
        from . import _lib
        from .api import _check
        _check(_lib.lib().mumode_comm_set_exchange(self.c, {"nccl": 0, "p2p": 1}[mode]))

    def set_overlap_sms(self, sms: int) -> None:
        """SMs left to NCCL while sub-slabs overlap the exchange (default 16)."""
        from . import _lib
        from .api import _check
        _check(_lib.lib().mumode_comm_set_overlap_sms(self.c, int(sms)))

    def close(self) -> None:
        if getattr(self, "c", None):
            from . import _lib
            _lib.lib().mumode_comm_destroy(self.c)
            self.c = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def slab_plan_offsets(P: int, m: Sequence[int], n: Sequence[int]) -> tuple[list[int], list[int]]:
    """(c_off, a_off) from the C-ABI's mumode_slab_plan (host only)."""
    import ctypes

    from . import _lib
    from .api import _check
    c_off = (ctypes.c_int64 * (P + 1))()
    a_off = (ctypes.c_int64 * (P + 1))()
    _check(_lib.lib().mumode_slab_plan(int(P), len(m), _lib.i64_array(m), _lib.i64_array(n), c_off, a_off))
    return list(c_off), list(a_off)


def dist_plan(P: int, rank: int, m: Sequence[int], n: Sequence[int], chunks: int = 0, cplx: bool = False):
    """The exact schedule ``mumode_dist_tucker_*`` runs on ``rank`` (host-only
    C-ABI ``mumode_dist_plan``): ([(col0, width, send_off)] per sub-slab,
    [(chunk, kind, peer, send_off, z_off, count)] with kind 0 send, 1 receive,
    2 own-block copy; offsets and counts in doubles)."""
    import ctypes

    from . import _lib
    from .api import _check
    lib = _lib.lib()
    nc, no = ctypes.c_int(), ctypes.c_int()
    args = (int(P), int(rank), len(m), _lib.i64_array(m), _lib.i64_array(n), int(chunks), int(cplx))
    rc = lib.mumode_dist_plan(*args, None, 0, ctypes.byref(nc), None, 0, ctypes.byref(no))
    if rc != 0 and nc.value == 0 and no.value == 0:
        _check(rc)
    ct = (ctypes.c_int64 * max(1, 3 * nc.value))()
    ot = (ctypes.c_int64 * max(1, 6 * no.value))()
    _check(lib.mumode_dist_plan(*args, ct, nc.value, ctypes.byref(nc), ot, no.value, ctypes.byref(no)))
    chunks_ = [tuple(ct[3 * j:3 * j + 3]) for j in range(nc.value)]
    ops = [tuple(ot[6 * k:6 * k + 6]) for k in range(no.value)]
    return chunks_, ops


def dist_tucker(comm: Comm, T_local, Ls, m: Sequence[int], n: Sequence[int] | None = None, chunks: int = 4,
                out=None, phase: int | None = None):
    """One slab-partitioned Tucker application through the C-ABI
    (``mumode_dist_tucker_{f64,c128}``). ``T_local``: this rank's column-major
    last-mode slab on its GPU; ``Ls``: all d factors on the same GPU; ``m``,
    ``n``: GLOBAL extents. Returns this rank's (A_r x n_d) rows of the result as
    a flat column-major tensor (``gather_rows`` reassembles). ``phase`` (peer
    stores only): 1 = local modes + stores + signal, 2 = wait + last mode
    (``mumode_dist_tucker_phase_*``)."""
    import torch

    from . import _lib
    from .api import _check, get_handle, is_colmajor
    d = len(m)
    n = [int(L.shape[0]) for L in Ls] if n is None else [int(e) for e in n]
    cplx = T_local.is_complex() or any(L.is_complex() for L in Ls)
    dt = torch.complex128 if cplx else torch.float64
    if T_local.dtype != dt or not is_colmajor(T_local):
        raise ValueError("dist_tucker: T_local must be a column-major float64/complex128 slab "
                         "(complex factors need a complex slab)")
    Ls = [L.to(dt) for L in Ls]
    Ls = [L if is_colmajor(L) else L.t().contiguous().t() for L in Ls]
    c_off, a_off = slab_plan_offsets(comm.nranks, m, n)
    A_r = a_off[comm.rank + 1] - a_off[comm.rank]
    S = out if out is not None else torch.empty(A_r * n[-1], dtype=dt, device=T_local.device)
    h = get_handle(T_local.device.index)
    h.bind_torch_stream()
    if phase is None:
        fn = _lib.lib().mumode_dist_tucker_c128 if cplx else _lib.lib().mumode_dist_tucker_f64
        _check(fn(h.h, comm.c, d, _lib.i64_array(m), _lib.i64_array(n), T_local.data_ptr(),
                  _lib.ptr_array([L.data_ptr() for L in Ls]), S.data_ptr(), int(chunks)))
    else:
        fn = _lib.lib().mumode_dist_tucker_phase_c128 if cplx else _lib.lib().mumode_dist_tucker_phase_f64
        _check(fn(h.h, comm.c, d, _lib.i64_array(m), _lib.i64_array(n), T_local.data_ptr(),
                  _lib.ptr_array([L.data_ptr() for L in Ls]), S.data_ptr(), int(phase)))
    return S


def dist_return_plan(P: int, rank: int, n: Sequence[int]):
    """Schedule of the return exchange (host-only C-ABI mumode_dist_return_plan):
    [(0, kind, peer, rows_off, stage_off, count)]."""
    import ctypes

    from . import _lib
    from .api import _check
    lib = _lib.lib()
    no = ctypes.c_int()
    args = (int(P), int(rank), len(n), _lib.i64_array(n))
    rc = lib.mumode_dist_return_plan(*args, None, 0, ctypes.byref(no))
    if rc != 0 and no.value == 0:
        _check(rc)
    ot = (ctypes.c_int64 * max(1, 6 * no.value))()
    _check(lib.mumode_dist_return_plan(*args, ot, no.value, ctypes.byref(no)))
    return [tuple(ot[6 * k:6 * k + 6]) for k in range(no.value)]


def dist_expint(comm: Comm, u0_local, Es, m: Sequence[int], steps: int, out=None):
    """``steps`` exponential-integrator steps across ranks through the C-ABI
    (``mumode_dist_expint_f64``); ``u0_local`` / result: this rank's
    column-major last-mode slab."""
    import torch

    from . import _lib
    from .api import _check, get_handle, is_colmajor
    if u0_local.dtype != torch.float64 or not is_colmajor(u0_local):
        raise ValueError("dist_expint: u0_local must be a column-major float64 slab")
    Es = [E.to(torch.float64) for E in Es]
    Es = [E if is_colmajor(E) else E.t().contiguous().t() for E in Es]
    u = out if out is not None else torch.empty_like(u0_local)
    h = get_handle(u0_local.device.index)
    h.bind_torch_stream()
    _check(_lib.lib().mumode_dist_expint_f64(h.h, comm.c, len(m), _lib.i64_array(m),
                                            _lib.ptr_array([E.data_ptr() for E in Es]), u0_local.data_ptr(),
                                            u.data_ptr(), int(steps)))
    return u


def gather_rows(plan: SlabPlan, blocks: Sequence[np.ndarray]) -> np.ndarray:
    """Reassemble the full column-major result from the per-rank (A_r x n_d)
    row blocks (flat column-major arrays)."""
    n_d = plan.n[-1]
    cols = [np.asarray(b).reshape((plan.a_sizes[r], n_d), order="F") for r, b in enumerate(blocks)]
    full = np.concatenate(cols, axis=0)  # (A x n_d)
    return full.reshape(plan.n, order="F")


def scatter_slabs(plan: SlabPlan, T: np.ndarray) -> list[np.ndarray]:
    """Split a full column-major tensor into the per-rank last-mode slabs."""
    return [np.asfortranarray(T[..., plan.c_off[r]:plan.c_off[r + 1]]) for r in range(plan.P)]
