"""C4 (complex 128^3 -> 192^3) repeated: GPU runs against each other (bitwise)
and against the reference library and the C port, to localise an
intermittent mismatch."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle as O  # noqa: E402
import paper_2112_11238_b200 as mm  # noqa: E402

g = mm.Rng(1234)
T = g.normal((128, 128, 128), True)
Ls = [g.normal((192, 128), True) for _ in range(3)]
ref = O.ref_tucker(T, Ls)
port = O.port_tucker(T, Ls)
print("ref vs port", O.rel_fro(ref, port), flush=True)
dT = torch.from_numpy(np.asfortranarray(T)).cuda()
dL = [torch.from_numpy(np.asfortranarray(L)).cuda() for L in Ls]
first = None
for r in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    S = mm.tucker(dT, dL).cpu().numpy()
    if first is None:
        first = S
    e_ref, e_port = O.rel_fro(S, ref), O.rel_fro(S, port)
    same = np.array_equal(S, first)
    bad = np.argwhere(np.abs(S - port) > 1e-8 * np.abs(port).max())
    print(f"rep {r}: vs ref {e_ref:.2e} vs port {e_port:.2e} same-as-first {same} bad {len(bad)}"
          + (f" first bad {bad[0].tolist()} last {bad[-1].tolist()}" if len(bad) else ""), flush=True)
