"""GPU time of itucker on n^3 (real), per policy: 0 = auto (right-looking sweep kernel), 24 = without its 96-fibre tiles, 23 = left-looking.
python tools/itucker_time.py [n ...]"""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2112_11238_b200 as mm

ns = [int(a) for a in sys.argv[1:]] or [200]
h = mm.get_handle(0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device='cuda')
for n in ns:
    rng = np.random.default_rng(n)
    T = torch.from_numpy(np.asfortranarray(rng.standard_normal((n, n, n)))).cuda()
    T = mm.to_colmajor(T)
    F = mm.FactorizedStack([rng.standard_normal((n, n)) + 3.0 * np.eye(n) for _ in range(3)])
    res = {}
    for pol in (23, 24, 0):
        h.set_kernel_policy(pol)
        for _ in range(2):
            out = mm.itucker(T, F)
        ts = []
        for _ in range(7):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); out = mm.itucker(T, F); b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res[pol] = (float(np.median(ts)), out.clone())
    h.set_kernel_policy(0)
    roof = 3 * 2.0 * n ** 4 / 37.0e12 * 1e3
    same = bool(torch.equal(res[0][1], res[23][1])) and bool(torch.equal(res[24][1], res[23][1]))
    print(f"n={n}: left-looking {res[23][0]:.4f} ms, right-looking with 64-fibre tiles {res[24][0]:.4f} ms, auto {res[0][0]:.4f} ms "
          f"({100 * roof / res[0][0]:.1f} % of the mode-product roofline), bitwise equal: {same}", flush=True)
