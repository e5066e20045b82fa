"""Time each fused two-mode pass of C5 (24^6) separately: modes (1,2), (3,4),
(5,6) through mumode_tucker_range_f64."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402
from paper_2112_11238_b200 import _lib  # noqa: E402

lib = _lib.lib()
h = mm.get_handle(0)
h.bind_torch_stream()
policy = int(sys.argv[1]) if len(sys.argv) > 1 else 0
h.set_kernel_policy(policy)
shape = (24,) * 6
T = mm.colmajor_empty(shape, torch.float64, "cuda").normal_()
S = torch.empty_like(T)
Ls = [mm.to_colmajor(torch.randn(24, 24, dtype=torch.float64, device="cuda")) for _ in range(6)]
P = _lib.ptr_array([L.data_ptr() for L in Ls])
m = _lib.i64_array(shape)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for lo in (1, 3, 5):
    ts = []
    for r in range(8):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rc = lib.mumode_tucker_range_f64(h.h, 6, m, m, T.data_ptr(), P, S.data_ptr(), lo, lo + 1)
        b.record()
        assert rc == 0
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    gb = 2 * T.numel() * 8 / 1e9
    print(f"policy {policy} pass modes {lo},{lo+1}: {ts[len(ts)//2]*1e3:.1f} us  -> {gb / (ts[len(ts)//2]*1e-3):.0f} GB/s")
