import torch, sys
sys.path.insert(0, '/root/repo')
import paper_2112_11238_b200 as mm
from paper_2112_11238_b200 import _lib
from paper_2112_11238_b200.dist import even_splits, offsets
lib, h = _lib.lib(), mm.get_handle(0); h.bind_torch_stream()
for A, C, P in [(65536, 32, 8), (65536, 128, 2), (40000, 200, 8)]:
    a_off = _lib.i64_array(offsets(even_splits(A, P)))
    Y = torch.randn(A * C, dtype=torch.float64, device="cuda"); S = torch.empty_like(Y)
    for _ in range(3): lib.mumode_slab_pack_f64(h.h, A, C, P, a_off, Y.data_ptr(), S.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): lib.mumode_slab_pack_f64(h.h, A, C, P, a_off, Y.data_ptr(), S.data_ptr())
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20
    print(f"pack A={A} C={C} P={P}: {t*1e3:.1f} us  {2*A*C*8/(t*1e-3)/1e9:.0f} GB/s")
