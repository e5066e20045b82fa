"""In-place block passes (block.cuh, policy 16) against the per-mode skinny path
(policy 14) and auto (policy 0): bitwise equality and Tucker GPU time, L2 flushed,
median of 10; roofline at 37.0 TF/s fp64 and 6553.6 GB/s."""
import sys, json
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import paper_2112_11238_b200 as mm

h = mm.get_handle(0)


def flops(m):
    return sum(2 * m[mu] * np.prod(m) for mu in range(len(m)))


flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device='cuda')
shapes = [tuple(int(x) for x in a.split('x')) for a in sys.argv[1:]] or \
    [(18,) * 6, (20,) * 6, (12,) * 6, (14,) * 6, (16,) * 6, (18, 14, 16, 10, 12, 22), (22,) * 5]
for m in shapes:
    torch.manual_seed(sum(m))
    T = mm.colmajor_empty(m, torch.float64, 'cuda').normal_()
    Ls = [mm.to_colmajor(torch.randn(e, e, dtype=torch.float64, device='cuda')) for e in m]
    res, outs = {}, {}
    for pol in (14, 16, 17, 0):
        h.set_kernel_policy(pol)
        outs[pol] = mm.tucker(T, Ls).clone()
        for _ in range(3):
            mm.tucker(T, Ls)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            mm.tucker(T, Ls)
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        res[pol] = float(np.median([a.elapsed_time(b) for a, b in ts]))
    h.set_kernel_policy(0)
    roof = max(flops(m) / 37.0e12, 16 * np.prod(m) / 6553.6e9) * 1e3
    print(json.dumps({"shape": "x".join(map(str, m)), "block_ms": round(res[16], 4), "per_mode_ms": round(res[14], 4),
                      "auto_ms": round(res[0], 4), "no_block_ms": round(res[17], 4), "roof_ms": round(roof, 4), "frac_block": round(roof / res[16], 3),
                      "frac_auto": round(roof / res[0], 3), "bitwise_block_vs_per_mode": bool(torch.equal(outs[16], outs[14])),
                      "max_abs_diff": float((outs[16] - outs[14]).abs().max())}), flush=True)
    del T
