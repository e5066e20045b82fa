"""GPU time of kronsumv (real) on n^d under policy 26 (one pass per term) and auto, L2 flushed, median of 10. python tools/kronsumv_time.py 200 3 [256 3 ...]"""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2112_11238_b200 as mm

args = [int(a) for a in sys.argv[1:]] or [200, 3]
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device='cuda')
for n, d in zip(args[::2], args[1::2]):
    V = mm.colmajor_empty((n,) * d, torch.float64, 'cuda').normal_()
    As = [mm.to_colmajor(torch.randn(n, n, dtype=torch.float64, device='cuda')) for _ in range(d)]
    res = {}
    for pol in (26, 0):  # 26: one pass per term; 0: auto (terms 1-2 fused for small square modes, kron12.cuh)
        mm.get_handle(0).set_kernel_policy(pol)
        for _ in range(3):
            mm.kronsumv(V, As)
        ts = []
        for _ in range(10):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); mm.kronsumv(V, As); b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res[pol] = float(np.median(ts))
    ms = res[0]
    roof = d * 2.0 * n ** (d + 1) / 37.0e12 * 1e3
    print(f"kronsumv {n}^{d}: per-term passes {res[26]:.4f} ms, auto {ms:.4f} ms ({100 * roof / ms:.1f} % of the fp64 roofline)",
          flush=True)
