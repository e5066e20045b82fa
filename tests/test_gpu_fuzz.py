"""Seeded fuzz of the device path against the plain-C oracle.

Random orders 1..5 with random extents (1..40, including 1, primes and odd
values that exercise every kernel path: TMA/DMMA, LDG-staged DMMA, SIMT,
fused pairs, odd-extent staging), random output extents (contractions and
expansions), real and complex, forward and adjoint, under each kernel policy.
The reference's own small-case tolerance (1e-13, test_tucker_ops.cpp) applies.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2112_11238_b200 as mm  # noqa: E402

EXTENTS = [1, 2, 3, 5, 7, 8, 9, 13, 16, 17, 24, 31, 32, 37, 40]


def _case(rng):
    d = int(rng.integers(1, 6))
    cap = {1: 40, 2: 40, 3: 40, 4: 17, 5: 9}[d]
    pool = [e for e in EXTENTS if e <= cap]
    m = [int(rng.choice(pool)) for _ in range(d)]
    n = [int(rng.choice(pool)) for _ in range(d)]
    cplx = bool(rng.integers(0, 4) == 0)
    adjoint = bool(rng.integers(0, 3) == 0)
    return m, n, cplx, adjoint


def _rnd(rng, shape, cplx):
    x = rng.uniform(-1, 1, shape)
    if cplx:
        x = x + 1j * rng.uniform(-1, 1, shape)
    return np.asfortranarray(x)


@pytest.mark.parametrize("policy", [0, 1, 2, 7, 8, 9, 11, 12, 18, 19, 20, 21])
def test_fuzz_tucker_and_mode_products(policy):
    rng = np.random.default_rng(4242 + policy)
    h = mm.get_handle(0)
    h.set_kernel_policy(policy)
    try:
        for it in range(40):
            m, n, cplx, adjoint = _case(rng)
            T = _rnd(rng, m, cplx)
            # stored factors: n x m (forward) or m x n (adjoint: cttucker applies P^H)
            Ls = [_rnd(rng, (m[k], n[k]) if adjoint else (n[k], m[k]), cplx) for k in range(len(m))]
            dT = torch.from_numpy(T).cuda()
            dL = [torch.from_numpy(L).cuda() for L in Ls]
            S = (mm.cttucker(dT, dL) if adjoint else mm.tucker(dT, dL)).cpu().numpy()
            ref = O.port_tucker(T, Ls, adjoint=adjoint)
            assert S.shape == ref.shape
            err = O.rel_max(S, ref)
            assert err < 1e-13, (it, m, n, cplx, adjoint, err)
            if not adjoint:
                mu = int(rng.integers(1, len(m) + 1))
                Sm = mm.mode_product(dT, dL[mu - 1], mu).cpu().numpy()
                assert O.rel_max(Sm, O.port_mode_product(T, Ls[mu - 1], mu)) < 1e-13, (it, m, mu)
    finally:
        h.set_kernel_policy(0)


def test_fuzz_block_passes_bitwise():
    # in-place block passes (block.cuh) on random square small-extent chains:
    # policy 16 forces cubes / 32-a blocks wherever a plan exists (mixed even
    # and odd extents, partial last blocks, orders 4..6), bitwise against one
    # skinny / tile pass per mode (policy 14) and against the oracle
    rng = np.random.default_rng(9191)
    h = mm.get_handle(0)
    pool = [2, 3, 4, 6, 7, 8, 10, 12, 13, 14, 16, 18, 20, 22, 24]
    try:
        for it in range(24):
            d = int(rng.integers(4, 7))
            cap = {4: 24, 5: 16, 6: 10}[d]
            m = [int(rng.choice([e for e in pool if e <= cap])) for _ in range(d)]
            m[0] = m[0] + (m[0] & 1)  # cubes need an even leading extent
            T = _rnd(rng, m, False)
            Ls = [_rnd(rng, (e, e), False) for e in m]
            dT = torch.from_numpy(T).cuda()
            dL = [torch.from_numpy(L).cuda() for L in Ls]
            h.set_kernel_policy(14)
            per_mode = mm.tucker(dT, dL)
            h.set_kernel_policy(16)
            blk = mm.tucker(dT, dL)
            assert torch.equal(blk, per_mode), (it, m)
            assert O.rel_max(blk.cpu().numpy(), O.port_tucker(T, Ls)) < 1e-13, (it, m)
    finally:
        h.set_kernel_policy(0)
