"""PCIe copy rates on the box (pinned host memory, 128 MiB): H2D alone, D2H
alone, both at once on two streams, and chunked variants -- the bound of the
host-buffer (e2e) Tucker path."""
import torch

N = 128 * 1024 * 1024
h_in = torch.empty(N // 8, dtype=torch.float64).pin_memory()
h_out = torch.empty(N // 8, dtype=torch.float64).pin_memory()
d_in = torch.empty(N // 8, dtype=torch.float64, device="cuda")
d_out = torch.empty(N // 8, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def spans(chunks):
    step = N // 8 // chunks
    return [(i * step, (i + 1) * step) for i in range(chunks)]


def h2d(chunks=1):
    s1.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        for a, b in spans(chunks):
            d_in[a:b].copy_(h_in[a:b], non_blocking=True)


def d2h(chunks=1):
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2):
        for a, b in spans(chunks):
            h_out[a:b].copy_(d_out[a:b], non_blocking=True)


for ch in (1, 8, 32):
    t1 = timed(lambda: h2d(ch))
    t2 = timed(lambda: d2h(ch))
    t3 = timed(lambda: (h2d(ch), d2h(ch)))
    print(f"chunks {ch:3d}: H2D {N / t1 / 1e6:.1f} GB/s  D2H {N / t2 / 1e6:.1f} GB/s  "
          f"both {2 * N / t3 / 1e6:.1f} GB/s total ({t3:.3f} ms for 2 x 128 MiB)")
