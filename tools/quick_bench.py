"""Quick kernel timing of single mode products and the Tucker chain
(development aid; bench.py is the contract)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_11238_b200 as mm  # noqa: E402


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        a.record(s)
        fn()
        b.record(s)
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    return ts[len(ts) // 2]


def main():
    policy = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    h = mm.get_handle(0)
    h.set_kernel_policy(policy)
    cfgs = [((256, 256, 256), 256), ((200, 200, 200), 200), ((96, 512, 384), 128)]
    for shape, n in cfgs:
        T = mm.colmajor_empty(shape, torch.float64, "cuda").normal_()
        Ls = [torch.randn(n, e, dtype=torch.float64, device="cuda").t().contiguous().t() for e in shape]
        for mu in (1, 2, 3):
            ms = timeit(lambda: mm.mode_product(T, Ls[mu - 1], mu))
            numel = 1
            for e in shape:
                numel *= e
            flops = 2.0 * n * numel
            print(json.dumps({"shape": shape, "n": n, "mu": mu, "ms": round(ms, 4),
                              "tflops": round(flops / ms / 1e9, 2), "policy": policy}))
        ms = timeit(lambda: mm.tucker(T, Ls))
        flops, ext = 0.0, list(shape)
        for mu in range(3):
            numel = 1
            for e in ext:
                numel *= e
            flops += 2.0 * n * numel
            ext[mu] = n
        print(json.dumps({"shape": shape, "n": n, "tucker_ms": round(ms, 4), "tflops": round(flops / ms / 1e9, 2)}))


if __name__ == "__main__":
    main()
