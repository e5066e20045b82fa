"""Shared CUDA-event timing for the sweep tools: median of `reps` launches
after 3 warm-ups, device-resident inputs (no L2 flush: the sweeps compare
kernel choices on the same shape)."""
import torch


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in evs)[reps // 2]
