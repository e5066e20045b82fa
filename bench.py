#!/usr/bin/env python
"""Benchmark of the B200 mu-mode engine (driver contract).

Metric (BASELINE.json): Tucker operator fp64 GFLOP/s and % of roofline.
Workload at N=1: BASELINE configs[1] (C2) -- 3-D Tucker operator
S = T x_1 L_1 x_2 L_2 x_3 L_3, real fp64, T in R^{256^3}, L_mu 256 x 256, all
standard normal from the reference's generator (mt19937_64 seed 1234, tensor
then matrices). One step = one Tucker application (3 mode products,
2.577e10 flop). FLOP = sum_mu 2 n_mu (elements entering mode mu).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

* ``value``     device-resident throughput through the C-ABI
                (mumode_tucker_f64), CUDA events per step, L2 flushed between
                steps (256 MiB write, outside the events), max over ranks.
* ``e2e``       the same metric through the host drop-in entry point
                (mumode_host_tucker_f64) with pinned host buffers: H2D of T and
                the factors and D2H of S inside every timed step.
* ``roofline``  the dominant kernel (the TMA/DMMA mode-product kernel): its
                algorithmic flops per launch / its mean CUDA-event duration,
                against the fp64 tensor-pipe peak measured live (DMMA probe;
                MEASURED_PEAKS.json has no fp64 entry).
* ``cpu_baseline`` the reference library itself (oracle/_ref, compiled from the
                reference sources) on the host cores, same workload and bytes.

Multi-GPU (torchrun, N>1): the C2 tensor is slab-partitioned over the last
mode; see paper_2112_11238_b200/dist.py.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Tucker operator fp64 GFLOP/s and % of roofline at 1/2/4/8 B200 vs host CPU"
UNIT = "GFLOP/s"
SEED = 1234
C2 = (256, 256, 256)
PAPER_C2_GFLOPS = 115.0  # paper Fig. 1, tucker d=3 n=256, MATLAB on i7-8750H
WORKLOAD = "C2: 3-D Tucker operator fp64, T 256^3 (128 MiB), three 256x256 factors (BASELINE configs[1])"


def hbm_peak_gbs() -> float:
    """Measured copy bandwidth of this pool's B200s (MEASURED_PEAKS.json,
    driver-written); the profiling recipe's fallback when it is absent."""
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        return 6545.6


def tucker_flops(m, n):
    ext, f = list(m), 0.0
    for mu in range(len(m)):
        f += 2.0 * n[mu] * float(np.prod(ext))
        ext[mu] = n[mu]
    return f


# ----------------------------------------------------------------- clocks
# throttle reasons that invalidate a timed run (sw_power_cap is kept and noted)
THROTTLE_REJECT = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "hw_power_brake_slowdown"}


class ClockSampler:
    """nvidia-smi clocks line via NVML, sampled every 10 ms during the run."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device: int):
        self.samples = []
        self.reasons = 0
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                util = nv.nvmlDeviceGetUtilizationRates(self.h).gpu
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((mhz, util, r))
            except Exception:
                pass
            time.sleep(0.01)

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        loaded = [s for s in self.samples if s[1] > 0] or self.samples
        bits = 0
        for s in loaded:
            bits |= s[2]
        reasons = [name for bit, name in self.REASONS.items() if bits & bit and bit != 0x1]
        return {"sm_mhz": statistics.median(s[0] for s in loaded), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(loaded)}


# ----------------------------------------------------------------- reference arm
def run_reference(args, rank: int) -> None:
    """The driver's reference arm: the reference library itself (oracle/_ref,
    compiled from /root/reference/proj/src) on all host cores. One call into
    it draws the C2 inputs with the reference's generator and times each
    ops::tucker application in C++ (oracle/ref_shim.cpp ref_bench_tucker_f64),
    so neither this package nor any copy of the operands is on the path."""
    if rank != 0:
        return
    import oracle as O
    cores = os.cpu_count() or 1
    O.ref_lib(threads=cores)
    flops = tucker_flops(C2, [256, 256, 256])
    times, checksum = O.ref_bench_tucker(SEED, C2, (256, 256, 256), args.warmup, args.steps)
    total = float(sum(times))
    value = flops * args.steps / total / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * total / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": round(value / PAPER_C2_GFLOPS, 4), "dtype": "f64",
        "data": "synthetic (mt19937_64 seed 1234, standard normal, reference draw order)",
        "config": {"workload": WORKLOAD, "seed": SEED, "parallelism": "host CPU (OpenMP + OpenBLAS)"},
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"ops::tucker 256^3 x {args.steps} steps (full C2 workload per step), "
                                   f"reference library compiled from /root/reference/proj/src "
                                   f"(oracle/_ref), inputs drawn and each step timed inside it; "
                                   f"OpenBLAS {O.ref_blas_kernel_name()}"},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "result_checksum": checksum,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- our arm
_JSON_OUT = None  # the real stdout when library output is diverted (distributed runs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the C1/C3/C4/C5 side measurements")
    ap.add_argument("--force-dist", action="store_true", help="run the slab/NCCL path even at N=1 (testing)")
    ap.add_argument("--chunks", type=int, default=0,
                    help="N>1: sub-slabs per rank in mumode_dist_tucker_f64 (exchange of one overlaps the "
                         "next; 0 = auto)")
    ap.add_argument("--exchange", choices=["nccl", "p2p"], default="nccl",
                    help="N>1: NCCL grouped send/recv, or peer stores from the last local mode's epilogue")
    ap.add_argument("--overlap-sms", type=int, default=16,
                    help="N>1: SMs the compute leaves to NCCL while sub-slabs overlap the exchange")
    ap.add_argument("--py-dist", action="store_true",
                    help="N>1: the Python slab algorithm with a torch all-to-all instead of the C-ABI")
    ap.add_argument("--overlap", action="store_true", help="with --py-dist: chunked grouped send/recv")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist
    import paper_2112_11238_b200 as mm
    from paper_2112_11238_b200 import _lib

    torch.cuda.set_device(local)
    if world > 1 or args.force_dist:
        # rank 0's stdout carries exactly one JSON line: anything the
        # libraries print during the run (NCCL's "NCCL version ..." banner)
        # goes to stderr, the JSON line to the saved stdout
        global _JSON_OUT
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29561")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        run_distributed(args, world, rank, local)
        dist.destroy_process_group()
        return
    dev = torch.device("cuda", local)
    h = mm.get_handle(local)
    lib = _lib.lib()
    stream = torch.cuda.current_stream(dev)
    h.bind_stream(stream.cuda_stream)

    # ---- inputs (reference draw order), resident in HBM
    g = mm.Rng(SEED)
    T_host = g.normal(C2)
    L_host = [g.normal((256, 256)) for _ in range(3)]
    T = torch.from_numpy(T_host).to(dev)
    Ls = [torch.from_numpy(L).to(dev) for L in L_host]
    m = mm.api._lib.i64_array(C2)
    n = mm.api._lib.i64_array((256, 256, 256))
    S = mm.colmajor_empty(C2, torch.float64, dev)
    Lptr = _lib.ptr_array([L.data_ptr() for L in Ls])
    flops = tucker_flops(C2, [256, 256, 256])
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        rc = lib.mumode_tucker_f64(h.h, 3, m, n, T.data_ptr(), Lptr, S.data_ptr(), 0)
        if rc:
            raise RuntimeError(lib.mumode_last_error().decode())

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: exactly K steps; a run that saw thermal / hardware
    # slowdown is measured once more (the recipe's rejection rule)
    def timed_region():
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = h.launches
        for a, b in ev:
            flush.fill_(1.0)  # evict L2 between steps (outside the events)
            a.record(stream)
            step()
            b.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        return [a.elapsed_time(b) for a, b in ev], h.launches - l0

    step_ms, launches = timed_region()
    remeasured = False
    if set(clocks.summary().get("reasons", [])) & THROTTLE_REJECT:
        clocks.stop()
        clocks = ClockSampler(local)
        clocks.start()
        step_ms, launches = timed_region()
        remeasured = True
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = world * flops * args.steps / (total_ms * 1e-3) / 1e9

    # ---- roofline of the dominant kernel: per-launch events on the same stream
    mode_ms = []
    ext = list(C2)
    bufs = [T, mm.colmajor_empty(C2, torch.float64, dev), mm.colmajor_empty(C2, torch.float64, dev)]
    for _ in range(args.steps):
        flush.fill_(1.0)
        src = T
        for mu in (1, 2, 3):
            dst = bufs[1 + (mu % 2)]
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            rc = lib.mumode_mode_product_f64(h.h, 3, m, mu, 256, src.data_ptr(), Ls[mu - 1].data_ptr(), dst.data_ptr())
            b.record(stream)
            if rc:
                raise RuntimeError(lib.mumode_last_error().decode())
            mode_ms.append((a, b))
            src = dst
    torch.cuda.synchronize()
    launch_ms = statistics.mean(a.elapsed_time(b) for a, b in mode_ms)
    flops_per_launch = 2.0 * 256 * float(np.prod(ext))
    peak = ctypes_peak(lib, h)
    achieved_tf = flops_per_launch / (launch_ms * 1e-3) / 1e12
    clocks.stop()

    # ---- e2e through the host drop-in entry point, pinned buffers
    Tpin = torch.from_numpy(T_host).pin_memory()
    Lpin = [torch.from_numpy(L).pin_memory() for L in L_host]
    Spin = torch.empty(int(np.prod(C2)), dtype=torch.float64).pin_memory()
    Lhptr = _lib.ptr_array([L.data_ptr() for L in Lpin])

    def e2e_step():
        rc = lib.mumode_host_tucker_f64(h.h, 3, m, n, Tpin.data_ptr(), Lhptr, Spin.data_ptr(), 0)
        if rc:
            raise RuntimeError(lib.mumode_last_error().decode())

    for _ in range(args.steps):  # one untimed batch (see the async warm-up below)
        e2e_step()
    if world > 1:
        dist.barrier()
    # each e2e figure: the median of three (sync) / seven (async) batches of K applications (every
    # batch moves all of its inputs and results; one batch of ~0.1 s was at
    # the mercy of single host hiccups: 7.8-8.7 TFLOP/s across runs)
    sync_batches = []
    for _ in range(3):
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        sync_batches.append(time.perf_counter() - t0)
    e2e_sync_s = statistics.median(sync_batches)
    # the same K applications queued back to back through the async entry
    # point: step k's download overlaps step k+1's upload (every step still
    # moves its input H2D and its result D2H inside the timed region)
    Spins = [Spin, torch.empty_like(Spin).pin_memory()]

    def e2e_async(k):
        rc = lib.mumode_host_tucker_f64_async(h.h, 3, m, n, Tpin.data_ptr(), Lhptr, Spins[k % 2].data_ptr())
        if rc:
            raise RuntimeError(lib.mumode_last_error().decode())

    # warm-up: two untimed batches (the first ~3 batches after an idle GPU run
    # 3.1-3.3 ms per application, then 2.95 steadily: tools/e2e_chunks.py)
    for _ in range(2):
        for k in range(args.steps):
            e2e_async(k)
        lib.mumode_host_wait(h.h)
    if world > 1:
        dist.barrier()
    async_batches = []
    for _ in range(7):  # median of seven: one run measured 7.2 TFLOP/s with two of three batches disturbed
        t0 = time.perf_counter()
        for k in range(args.steps):
            e2e_async(k)
        if lib.mumode_host_wait(h.h):
            raise RuntimeError(lib.mumode_last_error().decode())
        async_batches.append(time.perf_counter() - t0)
    e2e_s = statistics.median(async_batches)
    if world > 1:
        t = torch.tensor([e2e_s, e2e_sync_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s, e2e_sync_s = float(t[0]), float(t[1])
    e2e_value = world * flops * args.steps / e2e_s / 1e9
    e2e_sync_value = world * flops * args.steps / e2e_sync_s / 1e9
    h2d = Tpin.numel() * 8 + sum(L.numel() * 8 for L in Lpin)
    d2h = Spin.numel() * 8

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    traffic = None
    prof = ROOT / "profiles" / "roofline_traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": round(value / PAPER_C2_GFLOPS, 3), "dtype": "f64",
        "data": "synthetic (mt19937_64 seed 1234, standard normal, reference draw order)",
        "config": {"workload": WORKLOAD, "seed": SEED,
                   "l2": "flushed between steps (256 MiB write outside the step events)",
                   "parallelism": "single GPU" if world == 1 else f"replicas x{world}",
                   "pct_fp64_roofline": round(100.0 * (flops / (peak * 1e12)) / (total_ms * 1e-3 / args.steps), 2),
                   "vs_baseline_source": "BASELINE.md: paper Fig.1 tucker d=3 n=256, 0.224 s = 115.0 GFLOP/s (MATLAB, i7-8750H)"},
        "roofline": {"bound": "tensor", "achieved": round(achieved_tf, 3), "peak": round(peak, 3),
                     "unit": "TFLOP/s", "frac": round(achieved_tf / peak, 4), "traffic": traffic,
                     "kernel": "modeprod_tma_kernel (TMA 64B-swizzle ring + DMMA.8x8x4)",
                     "flops_per_launch": flops_per_launch, "mean_launch_ms": round(launch_ms, 5),
                     "peak_source": "fp64 DMMA probe measured live in this run (mumode_probe_fp64_peak); "
                                    "MEASURED_PEAKS.json has no fp64 entry",
                     "peak_crosscheck": {"cublas_dgemm_8192_tflops": cublas_dgemm_tflops(dev),
                                         "nominal_tflops": 37.2,
                                         "note": "148 SM x 128 flop/clk x 1.965 GHz"}},
        "e2e": {"value": round(e2e_value, 3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "path": "median of 7 batches of mumode_host_tucker_f64_async x K + mumode_host_wait (host-buffer C-ABI), pinned "
                        "buffers: consecutive steps overlap download and upload",
                "batch_ms_per_step": [round(b / args.steps * 1e3, 4) for b in async_batches],
                "sync_value": round(e2e_sync_value, 3),
                "sync_path": "mumode_host_tucker_f64 per step (returns with the result in host memory)"},
        "gpu_launches": int(launches),
        "clocks": dict(clocks.summary(), remeasured=remeasured),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(flops)
    if world == 1 and not args.no_extras:
        line["extras"] = extras(mm, lib, h, dev, stream, peak, flush)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_distributed(args, world, rank, local):
    """C2 slab-partitioned over the last mode across `world` GPUs (strong
    scaling: the same 256^3 Tucker application, split) through the C-ABI
    mumode_dist_tucker_f64: per sub-slab local modes 1-2 + pack on the compute
    stream, grouped NCCL send/recv on the exchange stream (overlapping the next
    sub-slab), then local mode 3 (csrc/slab_dist.cuh). --py-dist runs the
    Python algorithm of paper_2112_11238_b200/dist.py with a torch all-to-all."""
    import torch
    import torch.distributed as dist
    import paper_2112_11238_b200 as mm
    from paper_2112_11238_b200 import _lib
    from paper_2112_11238_b200.dist import (Comm, CudaSlabBackend, SlabPlan, dist_tucker, scatter_slabs,
                                            slab_tucker, slab_tucker_overlapped)

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    h = mm.get_handle(local)
    lib = _lib.lib()
    stream = torch.cuda.current_stream(dev)
    h.bind_stream(stream.cuda_stream)
    g = mm.Rng(SEED)
    T_host = g.normal(C2)
    L_host = [g.normal((256, 256)) for _ in range(3)]
    plan = SlabPlan(C2, (256, 256, 256), world)
    T_r_host = scatter_slabs(plan, T_host)[rank]
    T_r = torch.from_numpy(T_r_host).to(dev)
    Ls = [torch.from_numpy(L).to(dev) for L in L_host]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    S_out = torch.empty(plan.a_sizes[rank] * 256, dtype=torch.float64, device=dev)
    if not args.py_dist:
        # the C-ABI path (own NCCL communicator); if it cannot come up the run
        # fails loudly -- the Python slab algorithm runs only when asked for
        comm = Comm.from_torch(device=local)
        comm.set_exchange(args.exchange)
        comm.set_overlap_sms(args.overlap_sms)
        dist_tucker(comm, T_r, Ls, C2, chunks=args.chunks, out=S_out)
        comm.poll(timeout_ms=120000)
    if args.py_dist:
        be = CudaSlabBackend(local)
        if args.overlap:
            def run_slab(T_in):
                return slab_tucker_overlapped(plan, rank, T_in, Ls, be, chunks=4)
        else:
            def run_slab(T_in):
                return slab_tucker(plan, rank, T_in, Ls, be)
        path = "python slab algorithm, torch " + ("grouped send/recv (4 chunks)" if args.overlap else "all-to-all")
    else:
        def run_slab(T_in):
            return dist_tucker(comm, T_in, Ls, C2, chunks=args.chunks, out=S_out)
        path = ("C-ABI mumode_dist_tucker_f64, peer stores from the mode-2 epilogue (NVLink, CUDA IPC)"
                if args.exchange == "p2p" else
                "C-ABI mumode_dist_tucker_f64, NCCL grouped send/recv, "
                + (f"{args.chunks} overlapped sub-slabs" if args.chunks else "auto sub-slabs"))
    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        run_slab(T_r)
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    l0 = h.launches
    for e0, e1 in ev:
        flush.fill_(1.0)
        e0.record(stream)
        run_slab(T_r)
        e1.record(stream)
    if not args.py_dist:
        comm.poll(timeout_ms=120000)  # NCCL async errors / a lost peer fail the run instead of hanging
    torch.cuda.synchronize()
    dist.barrier()
    launches = h.launches - l0
    total_ms = sum(e0.elapsed_time(e1) for e0, e1 in ev)
    # the dominant kernel alone: local modes 1-2 on this rank's slab
    Y = torch.empty(256 * 256 * plan.c_sizes[rank], dtype=torch.float64, device=dev)
    ext = _lib.i64_array(plan.local_in_extents(rank))
    nn = _lib.i64_array([256, 256, plan.c_sizes[rank]])
    P = _lib.ptr_array([L.data_ptr() for L in Ls])
    lev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    for _ in range(2):  # descriptors and workspace for this shape
        lib.mumode_tucker_range_f64(h.h, 3, ext, nn, T_r.data_ptr(), P, Y.data_ptr(), 1, 2)
    for e0, e1 in lev:
        flush.fill_(1.0)
        e0.record(stream)
        lib.mumode_tucker_range_f64(h.h, 3, ext, nn, T_r.data_ptr(), P, Y.data_ptr(), 1, 2)
        e1.record(stream)
    torch.cuda.synchronize()
    local_ms = sum(e0.elapsed_time(e1) for e0, e1 in lev)
    t = torch.tensor([total_ms, local_ms], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, local_ms = float(t[0]), float(t[1])
    value = plan.flops() * args.steps / (total_ms * 1e-3) / 1e9
    peak = ctypes_peak(lib, h)
    local_flops = 2.0 * 256 * 256 * 256 * plan.c_sizes[rank] * 2  # modes 1, 2 on the slab
    achieved_tf = local_flops / (local_ms / args.steps * 1e-3) / 1e12
    clocks.stop()
    # e2e: the rank's slab from pinned host memory, its result rows back
    T_pin = torch.from_numpy(T_r_host).pin_memory()
    out_pin = torch.empty(plan.a_sizes[rank] * 256, dtype=torch.float64).pin_memory()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        T_dev = T_pin.to(dev, non_blocking=True)
        S_r = run_slab(T_dev)
        out_pin.copy_(S_r, non_blocking=True)
        torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = plan.flops() * args.steps / float(t[0]) / 1e9
    extras = {}
    if not args.py_dist and not args.no_extras:
        extras["C5_6d_24_slab"] = dist_c5(args, world, rank, dev, comm, stream, flush)
    if not args.py_dist:
        comm.close()
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": round(value / PAPER_C2_GFLOPS, 3), "dtype": "f64",
        "data": "synthetic (mt19937_64 seed 1234, standard normal, reference draw order)",
        "config": {"workload": WORKLOAD, "seed": SEED,
                   "parallelism": f"slab x{world} (last mode): {path}",
                   "l2": "flushed between steps (256 MiB write outside the step events)",
                   "exchange_bytes_per_rank": plan.exchange_bytes(rank),
                   "local_ms_per_step": round(local_ms / args.steps, 4),
                   "pct_fp64_roofline_per_gpu": round(100.0 * value / world / (peak * 1e3), 2)},
        "roofline": {"bound": "tensor", "achieved": round(achieved_tf, 3), "peak": round(peak, 3),
                     "unit": "TFLOP/s", "frac": round(achieved_tf / peak, 4), "traffic": None,
                     "kernel": "modeprod_tma_kernel, local modes 1-2 on the rank's slab (timed alone)",
                     "peak_source": "fp64 DMMA probe measured live (mumode_probe_fp64_peak)"},
        "e2e": {"value": round(e2e_value, 3), "unit": UNIT, "h2d_bytes_per_step": int(T_pin.numel() * 8),
                "d2h_bytes_per_step": int(out_pin.numel() * 8),
                "path": "per rank: pinned slab H2D, slab-partitioned Tucker, result rows D2H"},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
    }
    if extras:
        line["extras"] = extras
    print(json.dumps(line), file=_JSON_OUT or sys.stdout, flush=True)


def dist_c5(args, world, rank, dev, comm, stream, flush):
    """BASELINE configs[4]: the 6-D 24^6 Tucker slab-partitioned over the last
    mode across the ranks (24/P columns each), through the same C-ABI path
    (fused local passes, exchange, last mode). Device-generated synthetic
    slab (no parity check here; tests cover the path)."""
    import torch
    import torch.distributed as dist
    import paper_2112_11238_b200 as mm
    from paper_2112_11238_b200.dist import SlabPlan, dist_tucker
    m = (24,) * 6
    plan = SlabPlan(m, m, world)
    gen = torch.Generator(device=dev).manual_seed(SEED + rank)
    T_r = torch.empty((24,) * 5 + (plan.c_sizes[rank],), dtype=torch.float64, device=dev)
    T_r = mm.to_colmajor(torch.randn(T_r.shape, dtype=torch.float64, device=dev, generator=gen))
    g = torch.Generator(device=dev).manual_seed(SEED)
    Ls = [mm.to_colmajor(torch.randn(24, 24, dtype=torch.float64, device=dev, generator=g)) for _ in range(6)]
    out = torch.empty(plan.a_sizes[rank] * 24, dtype=torch.float64, device=dev)
    steps = max(3, min(args.steps, 10))
    for _ in range(3):
        dist_tucker(comm, T_r, Ls, m, chunks=args.chunks, out=out)
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(steps)]
    dist.barrier()
    for e0, e1 in ev:
        flush.fill_(1.0)
        e0.record(stream)
        dist_tucker(comm, T_r, Ls, m, chunks=args.chunks, out=out)
        e1.record(stream)
    torch.cuda.synchronize()
    ms = sum(e0.elapsed_time(e1) for e0, e1 in ev) / steps
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    return {"ms": round(ms, 4), "gflops": round(plan.flops() / (ms * 1e-3) / 1e9, 2),
            "exchange_bytes_per_rank": plan.exchange_bytes(rank), "steps": steps,
            "scaling": "strong (the full 24^6 application split over the ranks)"}


def cublas_dgemm_tflops(dev) -> float | None:
    """cuBLAS DGEMM (torch float64 matmul) at 8192^3 on this GPU: a library
    yardstick printed beside the DMMA probe that is the roofline denominator."""
    import torch
    try:
        a = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
        b = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
        a @ b
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(5):
            e0.record()
            a @ b
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b
        return round(2 * 8192 ** 3 / (best * 1e-3) / 1e12, 3)
    except Exception:  # reported as unavailable, never replaces the probe
        return None


def ctypes_peak(lib, h) -> float:
    import ctypes
    v = ctypes.c_double()
    rc = lib.mumode_probe_fp64_peak(h.h, ctypes.byref(v))
    if rc:
        raise RuntimeError(lib.mumode_last_error().decode())
    return float(v.value)


def cpu_baseline(flops):
    """The reference library (oracle/_ref) on this box's host cores: the same
    C2 workload, inputs drawn inside it with the same generator and seed, each
    ops::tucker timed in C++ (the --impl reference arm's measurement, bounded
    to 1 warm-up + 5 steps)."""
    try:
        import oracle as O
        cores = os.cpu_count() or 1
        O.ref_lib(threads=cores)
        reps = 5
        times, _ = O.ref_bench_tucker(SEED, C2, (256, 256, 256), 1, reps)
        med = statistics.median(times)
        return {"value": round(flops / med / 1e9, 3), "unit": UNIT, "cores": cores, "kind": "reference",
                "sample": f"ops::tucker on the full C2 workload (256^3), 1 warm-up + median of {reps}; "
                          f"OMP/OpenBLAS threads = {cores}; OpenBLAS core {O.ref_blas_kernel_name()}",
                "seconds_per_step": round(med, 4)}
    except Exception as e:  # reported, never silently replaced
        return {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                "sample": f"unavailable: {e}"}


def extras(mm, lib, h, dev, stream, peak, flush):
    """Side measurements on the other BASELINE configs (device-resident,
    events, L2 flushed): GFLOP/s and fraction of the fp64 roofline."""
    import torch
    out = {}

    def timeit(fn, reps=10):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(reps):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            ts.append((a, b))
        torch.cuda.synchronize()
        return statistics.median(a.elapsed_time(b) for a, b in ts)

    def rec(name, flops, ms, bytes_alg):
        t_roof = max(flops / (peak * 1e12), bytes_alg / (hbm_peak_gbs() * 1e9))
        out[name] = {"ms": round(ms, 4), "gflops": round(flops / ms / 1e6, 2),
                     "roofline_frac": round(t_roof / (ms * 1e-3), 4)}

    def normal(shape, cplx=False):
        t = mm.colmajor_empty(shape, torch.complex128 if cplx else torch.float64, dev)
        return t.normal_()

    # C2 single modes
    T = normal((256, 256, 256))
    L = mm.to_colmajor(torch.randn(256, 256, dtype=torch.float64, device=dev))
    for mu in (1, 2, 3):
        ms = timeit(lambda: mm.mode_product(T, L, mu))
        rec(f"C2_mode{mu}", 2.0 * 256 * 256 ** 3, ms, 2 * 8 * 256 ** 3)
    # the reference CLI's bench-tucker (tools/mumode_cli.cpp:219-255): the fused
    # chain against tucker_sequential (standalone mode products, fresh
    # intermediates), with the CLI's <= 1e-12 agreement check
    L3 = [mm.to_colmajor(torch.randn(256, 256, dtype=torch.float64, device=dev)) for _ in range(3)]
    ms = timeit(lambda: mm.tucker_sequential(T, L3))
    rec("C2_tucker_sequential", tucker_flops((256,) * 3, (256,) * 3), ms, 2 * 8 * 256 ** 3)
    fused, seq = mm.tucker(T, L3), mm.tucker_sequential(T, L3)
    out["C2_tucker_sequential"]["fused_vs_sequential_rel_max"] = float(
        ((fused - seq).abs().max() / fused.abs().max()).item())
    # C1 2-D
    T1 = normal((100, 100))
    L1 = [mm.to_colmajor(torch.randn(100, 100, dtype=torch.float64, device=dev)) for _ in range(2)]
    ms = timeit(lambda: mm.tucker(T1, L1))
    rec("C1_2d_n100", tucker_flops((100, 100), (100, 100)), ms, 3 * 8 * 100 * 100 + 8 * 100 * 100)
    # C3: 100 exponential-integrator steps (one CUDA graph)
    A = torch.zeros(200, 200, dtype=torch.float64)
    hh = 1.0 / 201
    for i in range(200):
        A[i, i] = -2 / hh ** 2
        if i > 0:
            A[i, i - 1] = 1 / hh ** 2 - 0.5 / (2 * hh)
        if i < 199:
            A[i, i + 1] = 1 / hh ** 2 + 0.5 / (2 * hh)
    E = torch.from_numpy(mm.expm((1e-3 * A).numpy())).to(dev)
    u0 = normal((200, 200, 200))
    u1 = mm.colmajor_empty((200, 200, 200), torch.float64, dev)
    ms = timeit(lambda: mm.expint(u0, [E, E, E], 100, out=u1), reps=3)
    rec("C3_expint_200cube_100steps", 100 * tucker_flops((200,) * 3, (200,) * 3), ms, 100 * 2 * 8 * 200 ** 3)
    # C4 complex 128^3 -> 192^3
    Tc = normal((128, 128, 128), True)
    Lc = [mm.to_colmajor(torch.randn(192, 128, dtype=torch.complex128, device=dev)) for _ in range(3)]
    ms = timeit(lambda: mm.tucker(Tc, Lc))
    rec("C4_complex_128_to_192", 4 * tucker_flops((128,) * 3, (192,) * 3), ms, 16 * (128 ** 3 + 192 ** 3))
    # C5 6-D 24^6
    del T
    T5 = normal((24,) * 6)
    L5 = [mm.to_colmajor(torch.randn(24, 24, dtype=torch.float64, device=dev)) for _ in range(6)]
    ms = timeit(lambda: mm.tucker(T5, L5), reps=3)
    rec("C5_6d_24", tucker_flops((24,) * 6, (24,) * 6), ms, 2 * 8 * 24 ** 6)
    # the paper's own d = 6 sizes (n = 12..18) and 20^6:
    # cube passes of modes 1-3 + 32-a pair / skinny passes (block.cuh,
    # skinny.cuh); 16^6 takes the MU kernels (fused_ws / tail_ws)
    for n6 in (12, 14, 16, 18, 20):
        T6 = normal((n6,) * 6)
        L6 = [mm.to_colmajor(torch.randn(n6, n6, dtype=torch.float64, device=dev)) for _ in range(6)]
        ms = timeit(lambda: mm.tucker(T6, L6), reps=5)
        rec(f"d6_{n6}", tucker_flops((n6,) * 6, (n6,) * 6), ms, 2 * 8 * n6 ** 6)
        del T6
    # kronsumv (terms accumulated in the epilogues), itucker (per-mode
    # LU solves, 2 n^2 flop per fibre and mode) and the IMEX direct solve (two
    # Tuckers + divide) -- flops as the equivalent mode products, bytes compulsory
    ms = timeit(lambda: mm.kronsumv(T5, L5), reps=3)
    rec("kronsumv_6d_24", 6 * 2.0 * 24 * 24 ** 6, ms, 2 * 8 * 24 ** 6)
    del T5
    V3 = normal((200,) * 3)
    A3 = [mm.to_colmajor(torch.randn(200, 200, dtype=torch.float64, device=dev)) for _ in range(3)]
    ms = timeit(lambda: mm.kronsumv(V3, A3))
    rec("kronsumv_200cube", 3 * 2.0 * 200 * 200 ** 3, ms, 2 * 8 * 200 ** 3)
    F = mm.FactorizedStack([np.random.default_rng(k).standard_normal((200, 200)) + 30 * np.eye(200)
                            for k in range(3)])
    ms = timeit(lambda: mm.itucker(V3, F))
    rec("itucker_200cube", 3 * 2.0 * 200 * 200 ** 3, ms, 2 * 8 * 200 ** 3)
    An = A.numpy()
    M = (-1e-3) * (0.5 * (An + An.T)) + np.eye(200) / 3  # symmetric tridiagonal (the Laplacian part)
    solver = mm.KronSumSolver(Ms=[M, M, M])
    ms = timeit(lambda: solver.solve(V3))
    rec("imex_direct_solve_200cube", 2 * tucker_flops((200,) * 3, (200,) * 3), ms, 2 * 8 * 200 ** 3)
    return out


if __name__ == "__main__":
    main()
