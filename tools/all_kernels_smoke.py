"""Small cases that launch every kernel of the engine (TMA/DMMA real and
complex configs, LDG-staged, SIMT, fused pairs, tail, scatter / accumulate /
divide epilogues, pack / unpack, pad / staging, integrator graph, 1-rank dist
paths) and check each against the C oracle (test infrastructure only): a
quick whole-engine smoke for debugging on the GPU box.

  python tools/all_kernels_smoke.py"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle as O  # noqa: E402
import paper_2112_11238_b200 as mm  # noqa: E402
from paper_2112_11238_b200 import _lib  # noqa: E402
from paper_2112_11238_b200.dist import Comm, dist_expint, dist_tucker  # noqa: E402

rng = np.random.default_rng(0)
h = mm.get_handle(0)
lib = _lib.lib()


def rnd(shape, cplx=False):
    x = rng.standard_normal(shape)
    return np.asfortranarray(x + 1j * rng.standard_normal(shape) if cplx else x)


def check(S, ref, tol=1e-13, what=""):
    err = O.rel_max(S, ref)
    assert err < tol, (what, err)


def tucker_case(m, n, cplx=False, adjoint=False, policy=0):
    h.set_kernel_policy(policy)
    try:
        T = rnd(m, cplx)
        Ls = [rnd((m[k], n[k]) if adjoint else (n[k], m[k]), cplx) for k in range(len(m))]
        dT = torch.from_numpy(T).cuda()
        dL = [torch.from_numpy(L).cuda() for L in Ls]
        S = (mm.cttucker(dT, dL) if adjoint else mm.tucker(dT, dL)).cpu().numpy()
        check(S, O.port_tucker(T, Ls, adjoint=adjoint), what=(m, n, cplx, adjoint, policy))
    finally:
        h.set_kernel_policy(0)


# TMA/DMMA real: every forced configuration; complex: every complex config
for pol in (0, 3, 4, 5, 6):
    tucker_case((48, 40, 32), (40, 56, 24), policy=pol)
    tucker_case((24, 16, 40), (32, 24, 16), cplx=True, policy=pol)
tucker_case((40, 32, 24), (24, 40, 16), adjoint=True)           # materialised L^T
tucker_case((33, 17, 9), (21, 19, 7), policy=8)                  # LDG-staged
tucker_case((33, 17, 9), (21, 19, 7), cplx=True, policy=1)      # SIMT
tucker_case((24, 24, 24, 24), (24, 24, 24, 24))                  # fused pairs (FIRST + 16-wide)
tucker_case((8,) * 8, (8,) * 8)                                  # fused pairs + tail (A = 8^6)
tucker_case((24,) * 4, (24,) * 4, policy=9)                      # tail forced
tucker_case((209, 16, 16), (211, 16, 16))                        # L staging (odd n, mode 1 via LDG)
tucker_case((216, 210, 212), (209, 213, 210))                    # padded odd chain (all >= 208)

# kronsumv (accumulating epilogue), direct solver (divide epilogue)
V = rnd((32, 24, 16))
As = [rnd((e, e)) for e in V.shape]
W = mm.kronsumv(torch.from_numpy(V).cuda(), [torch.from_numpy(A).cuda() for A in As]).cpu().numpy()
ref = sum(O.port_mode_product(V, As[k], k + 1) for k in range(3))
check(W, ref, 1e-12, "kronsumv")
Ms = [np.eye(e) / 3 - 1e-2 * O.port_advection_diffusion(e, 0.0) for e in (40, 32, 24)]
solver = mm.KronSumSolver(Ms=Ms)
b = torch.from_numpy(rnd((40, 32, 24))).cuda()
x = solver.solve(b)
res = mm.kronsumv(x, [torch.from_numpy(M).cuda() for M in Ms]).cpu().numpy()
check(res, b.cpu().numpy(), 1e-12, "solve")

# integrator graph
E = torch.from_numpy(mm.expm(-1e-3 * O.port_advection_diffusion(24, 0.3))).cuda()
u0 = torch.from_numpy(rnd((24, 24, 24))).cuda()
u = mm.expint(u0, [E, E, E], 3).cpu().numpy()
ur = u0.cpu().numpy()
for _ in range(3):
    ur = O.port_tucker(ur, [E.cpu().numpy()] * 3)
check(u, ur, 1e-12, "expint")

# pack / unpack, scatter epilogue, dist paths (1 rank)
A, C, P = 1000, 7, 3
a_off = [0, 333, 334, 1000]
Y = torch.randn(A * C, dtype=torch.float64, device="cuda")
send, back = torch.empty_like(Y), torch.empty_like(Y)
assert lib.mumode_slab_pack_f64(h.h, A, C, P, _lib.i64_array(a_off), Y.data_ptr(), send.data_ptr()) == 0
assert lib.mumode_slab_unpack_f64(h.h, A, C, P, _lib.i64_array(a_off), send.data_ptr(), back.data_ptr()) == 0
assert torch.equal(back, Y)
m, n = (48, 40, 32), (40, 56, 24)
T = rnd(m)
Ls = [rnd((n[k], m[k])) for k in range(3)]
rows = 40 * 56
a_off = [0, 37, 37, 1121, rows]
bufs = [torch.zeros(max(1, (a_off[q + 1] - a_off[q]) * 32), dtype=torch.float64, device="cuda") for q in range(4)]
dT = torch.from_numpy(T).cuda()
dL = [torch.from_numpy(L).cuda() for L in Ls]
assert lib.mumode_tucker_range_scatter_f64(h.h, 3, _lib.i64_array(m), _lib.i64_array(n), dT.data_ptr(),
                                           _lib.ptr_array([L.data_ptr() for L in dL]), 1, 2, 4,
                                           _lib.i64_array(a_off), 0, _lib.ptr_array([b.data_ptr() for b in bufs])) == 0
for exch in ("nccl", "p2p"):
    comm = Comm(1, 0, Comm.unique_id(), 0)
    comm.set_exchange(exch)
    for chunks in (1, 3):
        S = dist_tucker(comm, dT, dL, m, n, chunks=chunks).cpu().numpy().reshape(n, order="F")
        check(S, O.port_tucker(T, Ls), what=("dist", exch, chunks))
    comm.close()
comm = Comm(1, 0, None, 0)
uu = dist_expint(comm, u0, [E, E, E], m=(24, 24, 24), steps=2).cpu().numpy()
comm.close()
torch.cuda.synchronize()
print("all kernels ok")
