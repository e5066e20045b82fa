"""Tucker GPU time of the d = 6 sizes n^6 (n = 12..24): auto (small-extent fused pairs
/ MU kernels) vs one mode per pass (policy 14), L2 flushed, median of 10; roofline at
37.0 TF/s fp64 and the measured HBM copy bandwidth."""
import sys, time, json
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import paper_2112_11238_b200 as mm
h = mm.get_handle(0)
def tf(m, n):
    ext=list(m); f=0
    for mu in range(len(m)):
        f += 2*n[mu]*np.prod(ext); ext[mu]=n[mu]
    return f
flush = torch.empty(64*1024*1024, dtype=torch.float32, device='cuda')
for e in [12, 14, 16, 18, 20, 22, 24]:
    m = (e,)*6
    T = mm.colmajor_empty(m, torch.float64, 'cuda').normal_()
    Ls = [mm.to_colmajor(torch.randn(e, e, dtype=torch.float64, device='cuda')) for _ in range(6)]
    res = {}
    for pol in (0, 14):
        h.set_kernel_policy(pol)
        for _ in range(3): mm.tucker(T, Ls)
        torch.cuda.synchronize()
        ts=[]
        for _ in range(10):
            flush.fill_(1.0)
            a,b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); mm.tucker(T, Ls); b.record(); ts.append((a,b))
        torch.cuda.synchronize()
        res[pol] = float(np.median([a.elapsed_time(b) for a,b in ts]))
    h.set_kernel_policy(0)
    flops = tf(m, m); byts = 16*e**6
    roof = max(flops/37.0e12, byts/6553.6e9)*1e3
    print(json.dumps({"n": e, "auto_ms": round(res[0],4), "per_mode_ms": round(res[14],4), "roof_ms": round(roof,4), "frac_auto": round(roof/res[0],3), "frac_per_mode": round(roof/res[14],3)}), flush=True)
    del T
