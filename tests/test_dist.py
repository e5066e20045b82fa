"""Slab-partitioned Tucker (paper_2112_11238_b200/dist.py).

CPU (no GPU): the partition / pack / all-to-all / assembly logic with
world_size 2 and 3 over gloo, local contractions by the CPU oracle (a test
backend that lives here -- the product has only the CUDA backend).
GPU: the CUDA backend's kernels (mumode_tucker_range_f64, mumode_slab_pack_f64,
the last-mode product) for P simulated ranks on one device with the exchange
emulated by slicing, and a real 1-rank NCCL group.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2112_11238_b200 as mm
from paper_2112_11238_b200.dist import (SlabPlan, gather_rows, scatter_slabs, slab_plan_offsets, slab_tucker,
                                        slab_tucker_overlapped)


class OracleGlooBackend:
    """Test backend: oracle (plain C restatement) for the local modes, numpy for
    the pack, gloo for the exchange."""

    def local_modes(self, T, m, n_all, Ls, lo, hi):
        cur = np.asfortranarray(np.asarray(T).reshape(m, order="F"))
        for mu in range(lo, hi + 1):
            cur = O.port_mode_product(cur, Ls[mu - 1], mu)
        return cur.reshape(-1, order="F")

    def pack(self, Y, A, C, a_off):
        Y2 = np.asarray(Y).reshape((A, C), order="F")
        return np.concatenate([Y2[a_off[q]:a_off[q + 1], :].reshape(-1, order="F") for q in range(len(a_off) - 1)])

    def alltoall(self, send, send_counts, recv_counts):
        out = torch.empty(sum(recv_counts), dtype=torch.float64)
        dist.all_to_all_single(out, torch.from_numpy(np.ascontiguousarray(send)), recv_counts, send_counts)
        return out.numpy()

    def last_mode(self, Z, rows, m_d, L_d):
        Z2 = np.asarray(Z).reshape((rows, m_d), order="F")
        return O.port_mode_product(Z2, L_d, 2).reshape(-1, order="F")

    # overlapped variant: torch CPU tensors as buffers, gloo point-to-point
    def empty(self, n):
        return torch.empty(n, dtype=torch.float64)

    def cols(self, T, rows_per_col, c0, w):
        return np.asarray(T).reshape(-1, order="F")[rows_per_col * c0: rows_per_col * (c0 + w)]

    def view(self, x, lo, hi):
        return x[lo:hi]

    def copy(self, dst, src):
        dst.copy_(torch.as_tensor(np.ascontiguousarray(src)))

    def post(self, sends, recvs):
        ops = [dist.P2POp(dist.isend, torch.as_tensor(np.ascontiguousarray(t)), p) for p, t in sends]
        ops += [dist.P2POp(dist.irecv, t, p) for p, t in recvs]
        return dist.batch_isend_irecv(ops)

    def wait(self, works):
        for w in works:
            w.wait()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for m, n, seed in cases:
            rng = np.random.default_rng(seed)
            T = np.asfortranarray(rng.standard_normal(m))
            Ls = [np.asfortranarray(rng.standard_normal((n[k], m[k]))) for k in range(len(m))]
            plan = SlabPlan(m, n, world)
            T_r = scatter_slabs(plan, T)[rank]
            S_r = slab_tucker(plan, rank, T_r, Ls, OracleGlooBackend())
            S_o = slab_tucker_overlapped(plan, rank, T_r, Ls, OracleGlooBackend(), chunks=3)
            blocks = [None] * world
            dist.all_gather_object(blocks, S_r)
            blocks_o = [None] * world
            dist.all_gather_object(blocks_o, np.asarray(S_o))
            if rank == 0:
                S = gather_rows(plan, blocks)
                So = gather_rows(plan, blocks_o)
                ref = O.port_tucker(T, Ls)
                q.put((m, n, max(O.rel_fro(S, ref), O.rel_fro(So, ref))))
    finally:
        dist.destroy_process_group()


CASES = [((6, 5, 4), (3, 7, 5), 1), ((4, 4, 4, 6), (4, 4, 4, 6), 2), ((7, 3, 9), (5, 4, 2), 3),
         ((5, 6), (8, 3), 4), ((2, 3, 2, 3, 4), (3, 2, 3, 2, 5), 5)]


@pytest.mark.parametrize("world", [2, 3])
def test_slab_tucker_gloo_matches_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    results = [q.get(timeout=30) for _ in CASES]
    for m, n, err in results:
        assert err < 1e-13, (m, n, err)


def test_plan_bookkeeping():
    plan = SlabPlan((256, 256, 256), (256, 256, 256), 8)
    assert plan.c_sizes == [32] * 8 and plan.A == 65536 and plan.a_sizes == [8192] * 8
    assert sum(plan.send_counts(3)) == 65536 * 32 == sum(plan.recv_counts(3))
    assert plan.exchange_bytes(0) == 7 * 8192 * 32 * 8  # 14.7 MB per rank on 8 GPUs
    uneven = SlabPlan((5, 7), (4, 3), 3)
    assert uneven.c_sizes == [3, 2, 2] and uneven.a_sizes == [2, 1, 1]
    with pytest.raises(ValueError):
        SlabPlan((4, 2), (4, 2), 3)


def test_c_abi_slab_plan_matches_python_plan():
    # mumode_slab_plan (host-only C-ABI) == SlabPlan, the partition the gloo
    # tests exercise, so both multi-GPU paths agree on who holds what
    from paper_2112_11238_b200.api import SizeError
    for m, n, P in [((256, 256, 256), (256, 256, 256), 8), ((5, 7), (4, 3), 3), ((24,) * 6, (24,) * 6, 8),
                    ((6, 5, 4), (3, 7, 5), 2), ((2, 3, 2, 3, 4), (3, 2, 3, 2, 5), 3), ((3, 64), (2, 64), 64)]:
        plan = SlabPlan(m, n, P)
        c_off, a_off = slab_plan_offsets(P, m, n)
        assert c_off == plan.c_off and a_off == plan.a_off, (m, n, P)
    with pytest.raises(SizeError, match="last mode extent 2 < 3 ranks"):
        slab_plan_offsets(3, (4, 2), (4, 2))


def _simulate_return(n, P, blocks):
    """Every rank executes its mumode_dist_return_plan schedule: output rows ->
    staging ([s][A_s x c_r]) -> slab (the slab_unpack_kernel mapping)."""
    from paper_2112_11238_b200.dist import dist_return_plan
    plan = SlabPlan(n, n, P)  # the output's own partition
    stages = [np.full(plan.A * plan.c_sizes[r], np.nan) for r in range(P)]
    from collections import defaultdict
    sq, rq = defaultdict(list), defaultdict(list)
    for r in range(P):
        for (_, kind, peer, boff, zoff, cnt) in dist_return_plan(P, r, n):
            if kind == 0:
                sq[(r, peer)].append((boff, cnt))
            elif kind == 1:
                rq[(peer, r)].append((zoff, cnt))
            else:
                stages[r][zoff:zoff + cnt] = blocks[r][boff:boff + cnt]
    assert set(sq) == set(rq)
    for (src, dst), lst in sq.items():
        assert len(lst) == len(rq[(src, dst)]) == 1
        (boff, cnt), (zoff, cnt2) = lst[0], rq[(src, dst)][0]
        assert cnt == cnt2
        assert np.isnan(stages[dst][zoff:zoff + cnt]).all()
        stages[dst][zoff:zoff + cnt] = blocks[src][boff:boff + cnt]
    slabs = []
    for r in range(P):
        assert not np.isnan(stages[r]).any()
        c_r = plan.c_sizes[r]
        Y = np.empty((plan.A, c_r))
        for q in range(P):
            lo, hi = plan.a_off[q], plan.a_off[q + 1]
            Y[lo:hi, :] = stages[r][lo * c_r: hi * c_r].reshape((hi - lo, c_r), order="F")
        slabs.append(Y.reshape(n[:-1] + (c_r,), order="F"))
    return slabs


def _simulate_tucker_blocks(T_slabs, Ls, m, n, P, chunks):
    """Row blocks of one slab-partitioned application (real) executed from the
    mumode_dist_plan schedules."""
    from paper_2112_11238_b200.dist import dist_plan
    d = len(m)
    plan = SlabPlan(m, n, P)
    A = plan.A
    sends, zs, sched = [], [], []
    for r in range(P):
        ch, ops = dist_plan(P, r, m, n, chunks, False)
        sched.append(ops)
        send = np.full(A * plan.c_sizes[r], np.nan)
        for col0, w, soff in ch:
            if w == 0:
                continue
            Y = np.asfortranarray(T_slabs[r][..., col0:col0 + w])
            for mu in range(1, d):
                Y = O.port_mode_product(Y, Ls[mu - 1], mu)
            Yd = Y.reshape((A, w), order="F")
            for q in range(P):
                lo, hi = plan.a_off[q], plan.a_off[q + 1]
                send[soff + lo * w: soff + hi * w] = Yd[lo:hi, :].reshape(-1, order="F")
        sends.append(send)
        zs.append(np.full(plan.a_sizes[r] * m[-1], np.nan))
    from collections import defaultdict
    sq, rq = defaultdict(list), defaultdict(list)
    for r, ops in enumerate(sched):
        for (j, kind, peer, boff, zoff, cnt) in ops:
            if kind == 0:
                sq[(r, peer)].append((j, boff, cnt))
            elif kind == 1:
                rq[(peer, r)].append((j, zoff, cnt))
            else:
                zs[r][zoff:zoff + cnt] = sends[r][boff:boff + cnt]
    for key in sq:
        for (j, boff, cnt), (j2, zoff, cnt2) in zip(sq[key], rq[key]):
            zs[key[1]][zoff:zoff + cnt] = sends[key[0]][boff:boff + cnt]
    return [O.port_mode_product(np.asfortranarray(zs[r].reshape((plan.a_sizes[r], m[-1]), order="F")), Ls[-1],
                                2).reshape(-1, order="F") for r in range(P)]


@pytest.mark.parametrize("P", [2, 3, 5])
def test_c_abi_return_exchange_and_two_integrator_steps_simulated(P):
    # mumode_dist_expint's step = dist_tucker schedule + return schedule +
    # unpack; two steps over P simulated ranks equal two oracle Tuckers
    for i, m in enumerate([(6, 5, 10), (4, 3, 4, 7), (9, 11)]):
        rng = np.random.default_rng(10 * P + i)
        u0 = np.asfortranarray(rng.standard_normal(m))
        Es = [np.asfortranarray(rng.standard_normal((e, e)) / e) for e in m]
        plan = SlabPlan(m, m, P)
        slabs = scatter_slabs(plan, u0)
        ref = u0
        for step in range(2):
            blocks = _simulate_tucker_blocks(slabs, Es, m, m, P, 2)
            slabs = _simulate_return(m, P, blocks)
            ref = O.port_tucker(ref, Es)
            assert O.rel_fro(np.concatenate(slabs, axis=-1), ref) < 1e-13, (m, P, step)


def _simulate_c_schedule(m, n, P, chunks, cplx, seed):
    """Every rank executes its mumode_dist_plan schedule on numpy buffers:
    local modes per sub-slab (oracle), the slab_pack layout, sends matched to
    receives in NCCL order per peer pair, own-block copies, then the last
    mode. Returns the relative error against the oracle Tucker."""
    from paper_2112_11238_b200.dist import dist_plan
    rng = np.random.default_rng(seed)

    def rnd(shape):
        x = rng.standard_normal(shape)
        return np.asfortranarray(x + 1j * rng.standard_normal(shape) if cplx else x)
    d = len(m)
    T = rnd(m)
    Ls = [rnd((n[k], m[k])) for k in range(d)]
    plan = SlabPlan(m, n, P)
    el = 2 if cplx else 1
    A = plan.A
    slabs = scatter_slabs(plan, T)
    sends, zs, sched = [], [], []
    for r in range(P):
        ch, ops = dist_plan(P, r, m, n, chunks, cplx)
        sched.append((ch, ops))
        send = np.full(A * plan.c_sizes[r] * el, np.nan)
        for col0, w, soff in ch:
            if w == 0:
                continue
            Tj = np.asfortranarray(slabs[r][..., col0:col0 + w])
            Y = Tj
            for mu in range(1, d):
                Y = O.port_mode_product(Y, Ls[mu - 1], mu)
            Yd = Y.reshape((A, w), order="F")
            Yd = np.stack([Yd.real, Yd.imag], axis=0).transpose(1, 0, 2).reshape(A * el, w) if cplx else Yd
            for q in range(P):  # slab_pack_kernel layout
                lo, hi = plan.a_off[q] * el, plan.a_off[q + 1] * el
                blk = Yd[lo:hi, :].reshape(-1, order="F")
                send[soff + lo * w: soff + lo * w + blk.size] = blk
        sends.append(send)
        zs.append(np.full(plan.a_sizes[r] * m[-1] * el, np.nan))
    # exchange: per (chunk, sender, receiver) the k-th send pairs with the k-th receive
    from collections import defaultdict
    sq, rq = defaultdict(list), defaultdict(list)
    for r, (ch, ops) in enumerate(sched):
        for (j, kind, peer, boff, zoff, cnt) in ops:
            if kind == 0:
                sq[(r, peer)].append((j, boff, cnt))
            elif kind == 1:
                rq[(peer, r)].append((j, zoff, cnt))
            else:
                assert peer == r
                assert np.isnan(zs[r][zoff:zoff + cnt]).all(), "own block overlaps"
                zs[r][zoff:zoff + cnt] = sends[r][boff:boff + cnt]
    assert set(sq) == set(rq)
    for key in sq:
        assert len(sq[key]) == len(rq[key])
        for (j, boff, cnt), (j2, zoff, cnt2) in zip(sq[key], rq[key]):
            assert j == j2 and cnt == cnt2, (key, j, j2, cnt, cnt2)
            src, dst = key
            assert np.isnan(zs[dst][zoff:zoff + cnt]).all(), "receive regions overlap"
            zs[dst][zoff:zoff + cnt] = sends[src][boff:boff + cnt]
    blocks = []
    for r in range(P):
        assert not np.isnan(zs[r]).any(), "Z not fully written"
        Z = zs[r]
        if cplx:
            Z = Z[0::2] + 1j * Z[1::2]
        Zm = Z.reshape((plan.a_sizes[r], m[-1]), order="F")
        blocks.append(O.port_mode_product(np.asfortranarray(Zm), Ls[-1], 2).reshape(-1, order="F"))
    return O.rel_fro(gather_rows(plan, blocks), O.port_tucker(T, Ls))


@pytest.mark.parametrize("P", [2, 3, 5, 8])
def test_c_abi_dist_schedule_simulated_ranks(P):
    # the C++ multi-rank schedule (offsets, chunking, send/receive matching)
    # executed by P simulated ranks on CPU reproduces the Tucker operator
    cases = [((6, 5, 8), (3, 7, 5), False), ((4, 4, 4, 9), (4, 4, 4, 6), False), ((7, 3, 17), (5, 4, 2), True),
             ((5, 13), (8, 3), False), ((2, 3, 2, 3, 8), (3, 2, 3, 2, 5), True), ((3, 2, 11), (1, 1, 4), False)]
    for i, (m, n, cplx) in enumerate(cases):
        if m[-1] < P:
            continue
        for chunks in (0, 1, 2, 3, 16):
            err = _simulate_c_schedule(m, n, P, chunks, cplx, 1000 * P + i)
            assert err < 1e-13, (m, n, P, chunks, cplx, err)


def test_c_abi_dist_plan_auto_chunks_and_sizes():
    from paper_2112_11238_b200.dist import dist_plan
    # C2 on 2 ranks: slabs of 128 columns x 65536 rows -> 2 auto sub-slabs; 8 ranks -> 1
    ch, ops = dist_plan(2, 0, (256, 256, 256), (256, 256, 256))
    assert [w for _, w, _ in ch] == [64, 64]
    assert sum(c for (_, k, _, _, _, c) in ops if k == 0) == 65536 // 2 * 128  # half the rows leave
    ch, ops = dist_plan(8, 3, (256, 256, 256), (256, 256, 256))
    assert [w for _, w, _ in ch] == [32]
    assert sum(1 for o in ops if o[1] == 0) == 7 and sum(1 for o in ops if o[1] == 1) == 7


# ------------------------------------------------------------------ GPU
class SimulatedExchange:
    """Wraps the CUDA backend for P ranks simulated on one GPU: the exchange
    is emulated by slicing the other ranks' send buffers (no kernels wait on
    one another)."""

    def __init__(self, inner, plan):
        self.inner, self.plan = inner, plan
        self.sends = {}

    def run(self, T_slabs, Ls):
        plan, P = self.plan, self.plan.P
        d = len(plan.m)
        sends = []
        for r in range(P):
            Y = self.inner.local_modes(T_slabs[r], plan.local_in_extents(r), plan.n, Ls, 1, d - 1)
            sends.append(self.inner.pack(Y, plan.A, plan.c_sizes[r], plan.a_off))
        outs = []
        for r in range(P):
            parts = []
            for s in range(P):
                off = offsets_of(plan.send_counts(s))
                parts.append(sends[s][off[r]:off[r + 1]])
            recv = torch.cat(parts)
            outs.append(self.inner.last_mode(recv, plan.a_sizes[r], plan.m[-1], Ls[-1]))
        return outs


def offsets_of(counts):
    o = [0]
    for c in counts:
        o.append(o[-1] + c)
    return o


@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_slab_tucker_cuda_kernels_simulated_ranks(P):
    from paper_2112_11238_b200.dist import CudaSlabBackend
    assert torch.cuda.is_available()
    for m, n in [((64, 48, 40), (56, 48, 72)), ((24, 24, 24, 24), (24, 24, 24, 24))]:
        rng = np.random.default_rng(P)
        T = np.asfortranarray(rng.standard_normal(m))
        Ls = [np.asfortranarray(rng.standard_normal((n[k], m[k]))) for k in range(len(m))]
        plan = SlabPlan(m, n, P)
        slabs = [torch.from_numpy(s).cuda() for s in scatter_slabs(plan, T)]
        Lds = [torch.from_numpy(L).cuda() for L in Ls]
        outs = SimulatedExchange(CudaSlabBackend(0), plan).run(slabs, Lds)
        S = gather_rows(plan, [o.cpu().numpy() for o in outs])
        assert O.rel_fro(S, O.port_tucker(T, Ls)) < 1e-13


@pytest.mark.gpu
def test_slab_tucker_overlapped_nccl_single_rank():
    from paper_2112_11238_b200.dist import CudaSlabBackend
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(10)
        m, n = (48, 40, 32), (40, 56, 24)
        T = np.asfortranarray(rng.standard_normal(m))
        Ls = [np.asfortranarray(rng.standard_normal((n[k], m[k]))) for k in range(3)]
        plan = SlabPlan(m, n, 1)
        S_r = slab_tucker_overlapped(plan, 0, torch.from_numpy(T).cuda(),
                                     [torch.from_numpy(L).cuda() for L in Ls], CudaSlabBackend(0), chunks=4)
        S = gather_rows(plan, [S_r.cpu().numpy()])
        assert O.rel_fro(S, O.port_tucker(T, Ls)) < 1e-13
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_slab_tucker_nccl_single_rank():
    from paper_2112_11238_b200.dist import CudaSlabBackend
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(9)
        m = n = (48, 40, 32)
        T = np.asfortranarray(rng.standard_normal(m))
        Ls = [np.asfortranarray(rng.standard_normal((n[k], m[k]))) for k in range(3)]
        plan = SlabPlan(m, n, 1)
        S_r = slab_tucker(plan, 0, torch.from_numpy(T).cuda(), [torch.from_numpy(L).cuda() for L in Ls],
                          CudaSlabBackend(0))
        S = gather_rows(plan, [S_r.cpu().numpy()])
        assert O.rel_fro(S, O.port_tucker(T, Ls)) < 1e-13
    finally:
        dist.destroy_process_group()


DIST_CASES = [((48, 40, 32), (40, 56, 24), False), ((24, 24, 24, 24), (24, 24, 24, 24), False),
              ((16, 12, 10), (12, 14, 9), True), ((30, 7), (11, 13), False), ((64, 48, 40), (56, 48, 72), False)]


def _dist_case(comm, m, n, cplx, chunks, seed):
    from paper_2112_11238_b200.dist import dist_tucker
    rng = np.random.default_rng(seed)
    def rnd(shape):
        x = rng.standard_normal(shape)
        if cplx:
            x = x + 1j * rng.standard_normal(shape)
        return np.asfortranarray(x)
    T = rnd(m)
    Ls = [rnd((n[k], m[k])) for k in range(len(m))]
    plan = SlabPlan(m, n, 1)
    Td = torch.from_numpy(T).cuda()
    S_r = dist_tucker(comm, Td, [torch.from_numpy(L).cuda() for L in Ls], m, n, chunks=chunks)
    S = gather_rows(plan, [S_r.cpu().numpy()])
    return O.rel_fro(S, O.port_tucker(T, Ls))


@pytest.mark.gpu
def test_dist_tucker_c_abi_nccl_single_rank():
    # the C-ABI slab-partitioned Tucker with a real (1-rank) NCCL communicator:
    # chunked local modes, pack, grouped exchange stream, last mode
    from paper_2112_11238_b200.dist import Comm
    comm = Comm(1, 0, Comm.unique_id(), 0)
    try:
        for i, (m, n, cplx) in enumerate(DIST_CASES):
            for chunks in (1, 3, 8):
                assert _dist_case(comm, m, n, cplx, chunks, 100 + i) < 1e-14, (m, n, cplx, chunks)
    finally:
        comm.close()


@pytest.mark.gpu
def test_dist_tucker_c_abi_wrapped_single_rank_matches_tucker_bitwise():
    from paper_2112_11238_b200.dist import Comm, dist_tucker
    comm = Comm(1, 0, None, 0)
    try:
        assert _dist_case(comm, (40, 32, 24), (24, 40, 32), False, 2, 7) < 1e-14
        # 1 rank, 1 chunk: same kernels and accumulation order as tucker()
        g = mm.Rng(1234)
        T = torch.from_numpy(g.normal((96, 64, 48))).cuda()
        Ls = [torch.from_numpy(g.normal((64, e))).cuda() for e in (96, 64, 48)]
        S_r = dist_tucker(comm, T, Ls, (96, 64, 48), chunks=1)
        ref = mm.tucker(T, Ls)
        assert np.array_equal(S_r.cpu().numpy(), ref.cpu().numpy().reshape(-1, order="F"))
    finally:
        comm.close()


def test_multi_rank_comm_requires_nccl_id():
    from paper_2112_11238_b200.dist import Comm
    with pytest.raises(ValueError):
        Comm(2, 0, None, 0)


@pytest.mark.gpu
def test_dist_expint_c_abi_single_rank_matches_expint_bitwise():
    from paper_2112_11238_b200.dist import Comm, dist_expint
    comm = Comm(1, 0, Comm.unique_id(), 0)
    try:
        g = mm.Rng(77)
        for m in [(40, 32, 24), (24, 24, 24, 24)]:
            u0 = torch.from_numpy(g.normal(m)).cuda()
            Es = [torch.from_numpy(mm.expm(-1e-3 * np.diag(np.arange(1.0, e + 1)) + 1e-4 * g.normal((e, e)))).cuda()
                  for e in m]
            for steps in (0, 1, 4):
                u = dist_expint(comm, u0, Es, m, steps)
                ref = mm.expint(u0, Es, steps)
                assert torch.equal(u, ref), (m, steps)
    finally:
        comm.close()


@pytest.mark.gpu
def test_slab_pack_unpack_kernels_against_numpy():
    from paper_2112_11238_b200 import _lib
    from paper_2112_11238_b200.dist import even_splits, offsets
    lib, h = _lib.lib(), mm.get_handle(0)
    h.bind_torch_stream()
    for A, C, P in [(65536, 32, 8), (1000, 7, 3), (5, 9, 5), (40000, 25, 8), (7, 1, 1), (130, 64, 64)]:
        a_off = offsets(even_splits(A, P))
        Y = torch.randn(A * C, dtype=torch.float64, device="cuda")
        send = torch.full_like(Y, float("nan"))
        assert lib.mumode_slab_pack_f64(h.h, A, C, P, _lib.i64_array(a_off), Y.data_ptr(), send.data_ptr()) == 0
        Yn = Y.cpu().numpy().reshape((A, C), order="F")
        ref = np.concatenate([Yn[a_off[q]:a_off[q + 1], :].reshape(-1, order="F") for q in range(P)])
        np.testing.assert_array_equal(send.cpu().numpy(), ref)
        back = torch.full_like(Y, float("nan"))
        assert lib.mumode_slab_unpack_f64(h.h, A, C, P, _lib.i64_array(a_off), send.data_ptr(), back.data_ptr()) == 0
        assert torch.equal(back, Y)


@pytest.mark.gpu
@pytest.mark.parametrize("policy", [0, 8, 1])
def test_scatter_epilogue_to_rank_buffers(policy):
    # the fused exchange's epilogue (EPI 2), simulated with P destination
    # buffers on one GPU: rows a_off[q]..a_off[q+1] of the range's result land
    # in buffer q at column col0 + c; odd offsets split 16-B pairs and
    # misalign rows, one rank is empty. policy 8 / 1: compute + scatter-copy.
    from paper_2112_11238_b200 import _lib
    lib, h = _lib.lib(), mm.get_handle(0)
    h.bind_torch_stream()
    h.set_kernel_policy(policy)
    try:
        for m, n, lo, hi, cplx in [((48, 40, 32), (40, 56, 24), 1, 2, False), ((64, 48, 20), (56, 48, 20), 1, 2, False),
                                   ((40, 30), (64, 30), 1, 1, False), ((16, 16, 16, 16), (16, 16, 16, 16), 1, 3, False),
                                   ((24, 16, 20), (32, 24, 16), 1, 2, True), ((40, 12), (48, 12), 1, 1, True)]:
            rng = np.random.default_rng(sum(m))

            def rnd(shape):
                x = rng.standard_normal(shape)
                return np.asfortranarray(x + 1j * rng.standard_normal(shape) if cplx else x)
            T = rnd(m)
            Ls = [rnd((n[k], m[k])) for k in range(len(m))]
            Y = T
            for mu in range(lo, hi + 1):
                Y = O.port_mode_product(Y, Ls[mu - 1], mu)
            rows = int(np.prod(Y.shape[:hi]))
            cols = Y.size // rows
            Y2 = Y.reshape((rows, cols), order="F")
            cuts = sorted({0, 37, 101 % rows, rows // 2 + 1, rows})
            a_off = [0, 37, 37] + [c for c in cuts if c > 37]  # rank 1 empty
            P = len(a_off) - 1
            col0 = 3
            dt = torch.complex128 if cplx else torch.float64
            bufs = [torch.full(((a_off[q + 1] - a_off[q]) * (col0 + cols + 2),), float("nan"), dtype=dt,
                               device="cuda") for q in range(P)]
            Td = torch.from_numpy(T).cuda()
            Lds = [torch.from_numpy(L).cuda() for L in Ls]
            fn = lib.mumode_tucker_range_scatter_c128 if cplx else lib.mumode_tucker_range_scatter_f64
            rc = fn(
                h.h, len(m), _lib.i64_array(m), _lib.i64_array(n), Td.data_ptr(), _lib.ptr_array([L.data_ptr() for L in Lds]),
                lo, hi, P, _lib.i64_array(a_off), col0, _lib.ptr_array([b.data_ptr() if b.numel() else 0 for b in bufs]))
            assert rc == 0, lib.mumode_last_error()
            for q in range(P):
                r = a_off[q + 1] - a_off[q]
                got = bufs[q].cpu().numpy().reshape((r, col0 + cols + 2), order="F")
                assert np.isnan(got[:, :col0].real).all() and np.isnan(got[:, col0 + cols:].real).all()
                ref = Y2[a_off[q]:a_off[q + 1], :]
                if r:
                    assert O.rel_max(got[:, col0:col0 + cols], ref) < 1e-13, (m, q)
    finally:
        h.set_kernel_policy(0)


@pytest.mark.gpu
def test_dist_tucker_peer_store_exchange_single_rank():
    # exchange 1 at one rank: the scatter epilogue writes into the comm's
    # double-buffered Z (own pointer), then mode d; bitwise equal to tucker()
    from paper_2112_11238_b200.dist import Comm, dist_tucker
    comm = Comm(1, 0, Comm.unique_id(), 0)
    try:
        comm.set_exchange("p2p")
        g = mm.Rng(5)
        for m, n, cplx in [((96, 64, 48), (64, 96, 40), False), ((24, 24, 24, 24, 24), (24, 24, 24, 24, 24), False),
                           ((60, 40), (30, 50), False), ((32, 24, 16), (40, 24, 24), True)]:
            T = torch.from_numpy(g.normal(m, cplx)).cuda()
            Ls = [torch.from_numpy(g.normal((n[k], m[k]), cplx)).cuda() for k in range(len(m))]
            ref = mm.tucker(T, Ls).cpu().numpy().reshape(-1, order="F")
            for _ in range(3):  # both Z parities
                S_r = dist_tucker(comm, T, Ls, m, n)
                assert np.array_equal(S_r.cpu().numpy(), ref), m
    finally:
        comm.close()


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 3, 8])
def test_dist_local_pack_free_send_layout_simulated_ranks(P):
    # The NCCL path's local half on the GPU for P simulated ranks
    # (mumode_dist_local_f64: sub-slab chains whose last local mode scatters
    # the packed send blocks and the own block, no pack kernel), the NCCL
    # sends / receives of the plan emulated by device copies, then mode d:
    # bitwise equal to the single-GPU tucker().
    import ctypes
    from collections import defaultdict

    import paper_2112_11238_b200 as mm
    from paper_2112_11238_b200 import _lib
    from paper_2112_11238_b200.dist import dist_plan
    lib = _lib.lib()
    h = mm.get_handle(0)
    h.bind_torch_stream()
    for m, n, chunks in [((64, 48, 40), (56, 48, 72), 3), ((24, 24, 24, 24), (24, 24, 24, 24), 2),
                         ((40, 33, 17), (48, 31, 20), 1)]:
        if m[-1] < P:
            continue
        rng = np.random.default_rng(P + len(m))
        T = np.asfortranarray(rng.standard_normal(m))
        Ls = [np.asfortranarray(rng.standard_normal((n[k], m[k]))) for k in range(len(m))]
        want = mm.tucker(torch.from_numpy(T).cuda(), [torch.from_numpy(L).cuda() for L in Ls]).cpu().numpy()
        plan = SlabPlan(m, n, P)
        Lds = [torch.from_numpy(L).cuda() for L in Ls]
        Lp = _lib.ptr_array([L.data_ptr() for L in Lds])
        slabs = [torch.from_numpy(np.asfortranarray(s)).cuda() for s in scatter_slabs(plan, T)]
        sends, zs, sched = [], [], []
        for r in range(P):
            ch, ops = dist_plan(P, r, m, n, chunks)
            sched.append(ops)
            send = torch.full((plan.A * plan.c_sizes[r],), float("nan"), dtype=torch.float64, device="cuda")
            Z = torch.full((plan.a_sizes[r] * m[-1],), float("nan"), dtype=torch.float64, device="cuda")
            rc = lib.mumode_dist_local_f64(h.h, P, r, len(m), _lib.i64_array(m), _lib.i64_array(n),
                                           slabs[r].data_ptr(), Lp, send.data_ptr(), Z.data_ptr(), chunks)
            assert rc == 0, lib.mumode_last_error().decode()
            sends.append(send)
            zs.append(Z)
        torch.cuda.synchronize()
        sq, rq = defaultdict(list), defaultdict(list)
        for r, ops in enumerate(sched):
            for (j, kind, peer, boff, zoff, cnt) in ops:
                if kind == 0:
                    sq[(r, peer)].append((boff, cnt))
                elif kind == 1:
                    rq[(peer, r)].append((zoff, cnt))
        for key in sq:
            for (boff, cnt), (zoff, cnt2) in zip(sq[key], rq[key]):
                src, dst = key
                zs[dst][zoff:zoff + cnt].copy_(sends[src][boff:boff + cnt])
        rows = []
        for r in range(P):
            assert not torch.isnan(zs[r]).any(), "Z not fully written"
            Zm = zs[r].cpu().numpy().reshape((plan.a_sizes[r], m[-1]), order="F")
            rows.append(mm.mode_product(torch.from_numpy(np.asfortranarray(Zm)).cuda(), Lds[-1], 2)
                        .cpu().numpy().reshape(-1, order="F"))
        np.testing.assert_array_equal(gather_rows(plan, rows), want)
