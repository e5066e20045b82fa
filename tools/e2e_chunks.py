"""Host-buffer C2 Tucker through mumode_host_tucker_f64_async, K queued calls:
ms per application (best of 3). Used with kHostChunks (csrc/mumode_gpu.cu)
rebuilt at 1, 2, 3, 4, 8 for the chunk sweep quoted in DESIGN.md."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402
from paper_2112_11238_b200 import _lib  # noqa: E402

lib = _lib.lib()
h = mm.get_handle(0)
ext = (256, 256, 256)
m = _lib.i64_array(ext)
Tpin = torch.randn(int(np.prod(ext)), dtype=torch.float64).pin_memory()
Lpin = [torch.randn(256 * 256, dtype=torch.float64).pin_memory() for _ in range(3)]
Spins = [torch.empty_like(Tpin).pin_memory() for _ in range(2)]
Lp = _lib.ptr_array([L.data_ptr() for L in Lpin])
K = 30
for _ in range(2):
    res = []
    for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
        for k in range(2):
            assert lib.mumode_host_tucker_f64_async(h.h, 3, m, m, Tpin.data_ptr(), Lp, Spins[k % 2].data_ptr()) == 0
        lib.mumode_host_wait(h.h)
        t0 = time.perf_counter()
        for k in range(K):
            assert lib.mumode_host_tucker_f64_async(h.h, 3, m, m, Tpin.data_ptr(), Lp, Spins[k % 2].data_ptr()) == 0
        assert lib.mumode_host_wait(h.h) == 0
        res.append((time.perf_counter() - t0) / K * 1e3)
    print(f"{min(res):.3f} ms per application ({2.5769e10 / (min(res) * 1e-3) / 1e12:.2f} TF/s); all batches (ms): "
          + " ".join(f"{r:.3f}" for r in res), flush=True)
