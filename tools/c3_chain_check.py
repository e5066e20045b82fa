import sys, torch, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tools')
import oracle as O, paper_2112_11238_b200 as mm
from odd_modes import timeit
E = torch.from_numpy(mm.expm(1e-3 * O.port_advection_diffusion(200, 0.5))).cuda()
u0 = torch.from_numpy(mm.Rng(1234).normal((200, 200, 200))).cuda()
h = mm.get_handle(0)
res = {}
for pol in (0, 11, 0, 11):
    h.set_kernel_policy(pol)
    ms = timeit(lambda: mm.expint(u0, [E, E, E], 100), reps=5)
    res.setdefault(pol, []).append(ms)
    out = mm.expint(u0, [E, E, E], 100)
    res.setdefault(f"o{pol}", out)
h.set_kernel_policy(0)
print({k: v for k, v in res.items() if isinstance(k, int)}, "bitwise", torch.equal(res["o0"], res["o11"]))
