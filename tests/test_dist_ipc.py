"""The peer-store exchange of the slab-partitioned Tucker across PROCESSES.

P processes share the one GPU of this build, each a rank with its own CUDA
context, handle and communicator (``mumode_comm_create_local``: no NCCL --
the CUDA-IPC handles of the double-buffered Z and of the epoch flags travel
over a gloo group). Every application runs in two phases with a host barrier
between them:

  phase 1  local modes 1..d-1, the last local mode's epilogue storing every
           row straight into the owning rank's Z through the IPC mappings,
           then the system-scope release of this rank's epoch flag in every
           peer;
  barrier  (gloo) -- every rank's phase 1 has completed on the device;
  phase 2  the acquire-wait on the flags (already set, so it returns at once:
           no kernel ever waits on another process, which one GPU could not
           guarantee to co-schedule) and mode d on the local Z.

This exercises what a single-process test cannot: the IPC handle export /
import, stores into another process's allocations, the epoch flags and the
parity double-buffering over consecutive applications. The result rows of
every rank must be bitwise equal to the single-GPU ``tucker()``.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, m, n, cplx, iters):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch
    import torch.distributed as dist

    import paper_2112_11238_b200 as mm
    from paper_2112_11238_b200.dist import Comm, SlabPlan, dist_tucker, scatter_slabs

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    g = mm.Rng(2024)
    T = g.normal(m, complex_=cplx)
    Ls = [g.normal((n[k], m[k]), complex_=cplx) for k in range(len(m))]
    want = mm.tucker(T, Ls)  # the single-GPU engine (host drop-in path)
    plan = SlabPlan(m, n, world)
    a0, a1 = plan.a_off[rank], plan.a_off[rank + 1]
    want_rows = want.reshape(-1, n[-1], order="F")[a0:a1]
    comm = Comm.local(world, rank, 0)
    mine = comm.ipc_export(m, n, cplx)
    allh = [None] * world
    dist.all_gather_object(allh, mine)
    comm.ipc_import(m, n, allh, cplx)
    T_r = torch.from_numpy(np.asfortranarray(scatter_slabs(plan, T)[rank])).cuda()
    Ld = [torch.from_numpy(np.asfortranarray(L)).cuda() for L in Ls]
    for it in range(iters):
        out = dist_tucker(comm, T_r, Ld, m, n, phase=1)
        torch.cuda.synchronize()
        dist.barrier()  # every rank's stores and flags are complete
        out = dist_tucker(comm, T_r, Ld, m, n, out=out, phase=2)
        torch.cuda.synchronize()
        got = out.cpu().numpy().reshape((a1 - a0, n[-1]), order="F")
        if not np.array_equal(got, want_rows):
            raise AssertionError(f"rank {rank} iteration {it}: rows differ from tucker() "
                                 f"(max |diff| {np.max(np.abs(got - want_rows)):.3e})")
        dist.barrier()  # nobody starts the next phase 1 before all read their Z
    comm.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,m,n,cplx", [
    (2, (64, 48, 40), (56, 48, 72), False),
    (2, (32, 24, 16), (40, 24, 24), True),
    (3, (40, 33, 17), (48, 31, 20), False),
])
def test_peer_store_exchange_across_processes(world, m, n, cplx):
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a GPU")
    import torch.multiprocessing as tmp
    tmp.spawn(_rank_main, args=(world, _free_port(), m, n, cplx, 3), nprocs=world, join=True)
