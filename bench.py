#!/usr/bin/env python
"""bench.py — atomic-subdomain predictions/s of the distributed MFP (arXiv 2308.14258).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--iters T] [--impl ours|reference]

One STEP = one complete mfp_solve of the C5 workload (4097 x 4097 grid points,
m = 32, 65,025 subdomain predictions per iteration = 4 phases) for T fixed
iterations (tol = 0, parity mode), i.e. every row of SURVEY §8(a): init (a0),
T x [4 x (gather a1, embed a2, split expansion a3, hidden GEMM chain a4, head
a5, scatter a6), halo exchange a7], delta a8 after every 16th iteration (the
library evaluates delta every check_every = 16 iterations also in the fixed-
iteration parity mode; tol = 0 only disables the stop), final phase (a9).  N = 1: the whole domain on one B200.  N > 1 (torchrun): the same domain
on a Py x Px processor grid (1x2, 2x2, 2x4), NCCL halo exchange — strong scaling
(default).  --scaling weak: a 1024 x 2048-point block per GPU instead (1024x2048,
2048x2048, 2048x4096, 4096x4096 at N = 1, 2, 4, 8).

Extra legs on rank 0 after the timed region: e2e, the chain's roofline (CUDA events
on its stream), time-to-converge (W-rand SDNet, exact subsolver vs DST-I, fitted
SDNet vs the paper's MAE-0.05 rule), and at N = 1 the C3 batch sweep, the
boundary-IO HBM roofline past L2 and the fp64 oracle on the host cores.

value = UNIQUE predictions (T x 65,025) x K / max-over-ranks device time of the
K timed steps (CUDA events on the solve stream, L2 flushed between steps, outside
the events).  e2e = the same metric through mfp_solve with HOST g / u buffers
(H2D of g and D2H of the full field inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "atomic-subdomain predictions/sec and MFP time-to-converge at 1/2/4/8 B200"
GRIDS = {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}
NX = NY = 4096
PRED_PER_ITER = (2 * (NX // 32) - 1) * (2 * (NY // 32) - 1)   # 65,025
HIDDEN_FLOP_PER_ROW = 3 * 2 * 128 * 128                        # a4: three d x d GEMM rows


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--iters", type=int, default=64, help="MFP iterations per step (T)")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--precision", default="bf16", choices=["bf16", "fp16", "fp32"])
    p.add_argument("--no-converge", action="store_true")
    p.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                   help="strong: C5 (4097^2) at every N (default); weak: a 1024x2048 block per GPU")
    p.add_argument("--halo", default="nccl", choices=["nccl", "p2p", "put"],
                   help="halo transport for N > 1: grouped NCCL send/recv (default), the peer-memory "
                        "pack + pull kernels of mfp_p2p_open, or halo puts from the chain epilogue "
                        "(mfp_p2p_set_mode PUT) (NEXT-2; IPC handles all-gathered over the process group)")
    p.add_argument("--no-extras", action="store_true",
                   help="skip the legs after the timed region (e2e, sweep, boundary IO, CPU baseline): "
                        "used for the ncu launch list of the step")
    return p.parse_args()


# ------------------------------------------------------------------ d = 256 leg
def wide_leg(mfp, torch, stream, cfg, g_dev, u_dev, flush, ppi, peaks, T=16, steps=3, D=256, gelu=1,
             kernel="k_chain_tc2w (d = 256 hidden GEMM chain)", rank=0, comm=None,
             max_over_ranks=lambda x: x, barrier=lambda: None):
    """The same MFP with another SDNet variant — by default the wide SDNet (d = 256,
    SURVEY §8(b)/(d) "report both d values"); with cfg.precision = FP16X the
    accuracy mode: predictions/s over `steps` solves of T iterations (device
    events, L2 flushed between solves, outside the events) and the roofline of its
    chain (rows x 3 x 2 x d^2 FLOP per launch / the launch's event time).  At N > 1
    every rank runs it on its share (collective), value = whole-job predictions /
    max-over-ranks device time, so the scaling run carries the d = 256 curve too."""
    from mfp_inputs import random_weights
    mw = mfp.Mfp(cfg, mfp.make_net(d=D, gelu=gelu), random_weights(0, d=D), rank=rank, nccl_comm=comm,
                 stream=stream)
    for _ in range(2):
        mw.solve_device(g_dev, T, 0.0, u_dev)
    torch.cuda.synchronize()
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        with torch.cuda.stream(stream):
            flush.fill_(float(i))
            ev[i][0].record(stream)
        mw.solve_device(g_dev, T, 0.0, u_dev)
        with torch.cuda.stream(stream):
            ev[i][1].record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev))
    prof = mw.profile(4)
    chain_ms = prof.chain_ms_total / max(prof.chain_launches, 1)
    flop = prof.chain_rows / max(prof.chain_launches, 1) * 3 * 2 * D * D
    peak = peaks.get("bf16_tflops_sustained", 1400.0)
    achieved = flop / (chain_ms / 1000.0) / 1e12
    mw.close()
    burst = peaks.get("bf16_tflops", 1630.0)
    return {"d": D, "value": ppi * T * steps / (ms / 1000.0), "unit": "predictions/s",
            "ms_per_solve": ms / steps, "iters_per_solve": T,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "frac_vs_burst_peak": achieved / burst, "kernel": kernel,
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained",
                         "flop_per_launch": flop, "chain_ms_per_launch": chain_ms,
                         "chain_per_phase_ms": prof.ms_chain, "gather_embed_per_phase_ms": prof.ms_gather_embed,
                         "iteration_ms": prof.ms_per_iter}}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi-equivalent clock / throttle-reason sampling (NVML) during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.stop_ev = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self.stop_ev.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ reference arm (oracle)
def cpu_oracle_rate(target_s: float = 12.0):
    """The oracle (fp64 C, OpenMP) as it stands, on a bounded sample of C5: SDNet
    predictions of phase-0 subdomains from the initial lattice, one by one."""
    import oracle
    from mfp_inputs import gp_boundary, random_weights

    w = random_weights(0).astype(np.float64)
    cfg = oracle.MfpConfig(NX, NY)
    U = np.zeros((NY + 1, NX + 1))
    from mfp_inputs import boundary_points
    bp = boundary_points(NX, NY)
    U[bp[:, 1], bp[:, 0]] = gp_boundary(NX, NY, 0)
    anc = np.concatenate([oracle.anchors(NX, NY, c) for c in range(4)])
    n = 16
    t0 = time.perf_counter()
    oracle.predict_from_field(cfg, U, anc[:n], 0, w)
    dt = time.perf_counter() - t0
    n = int(min(len(anc), max(16, n * target_s / max(dt, 1e-3))))
    t0 = time.perf_counter()
    oracle.predict_from_field(cfg, U, anc[:n], 0, w)
    dt = time.perf_counter() - t0
    return n / dt, n, dt, oracle.num_threads()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def set_oracle_threads(n: int) -> None:
    """OpenMP thread count of the oracle's parallel regions (libgomp ICV of this thread)."""
    import ctypes
    ctypes.CDLL("libgomp.so.1").omp_set_num_threads(int(n))


def cpu_baseline_leg() -> dict:
    """The oracle as it stands on the box's host cores (BASELINE.md "CPU baseline
    plan"), bounded to ~25 s: (1) the metric's unit on a C5 sample with every
    core, 5 runs -> median / min / max; (2) the same with 1 thread, 3 runs;
    (3) exact-subsolver MFP solves to delta <= 1e-6 max|g| (c = 16) at C1 (65^2)
    and C2 (513^2), wall time and iterations."""
    import oracle
    from mfp_inputs import gp_boundary
    allc = oracle.num_threads()
    runs = [cpu_oracle_rate(target_s=2.0) for _ in range(5)]
    rates = [r[0] for r in runs]
    set_oracle_threads(1)
    try:
        one = [cpu_oracle_rate(target_s=1.0) for _ in range(3)]
    finally:
        set_oracle_threads(allc)
    conv = {}
    for name, n in (("C1_65x65", 64), ("C2_513x513", 512)):
        g = gp_boundary(n, n, 0).astype(np.float64)
        tol = 1e-6 * float(np.max(np.abs(g)))
        t0 = time.perf_counter()
        r = oracle.mfp_run(oracle.MfpConfig(n, n, subsolver="exact", check_every=16), g, 200000, tol=tol)
        conv[name] = {"seconds": time.perf_counter() - t0, "iterations": r.iterations, "tol": tol,
                      "subsolver": "exact discrete Laplace (fp64)", "threads": allc}
    return {"value": float(statistics.median(rates)), "unit": "predictions/s", "cores": allc, "kind": "oracle",
            "min": float(min(rates)), "max": float(max(rates)), "runs": len(rates),
            "sample": f"{runs[0][1]} C5 subdomain SDNet predictions from the initial lattice per run (fp64 "
                      f"oracle, exact-erf GELU, ~2 s per run); median of {len(rates)} runs",
            "cpu_model": cpu_model(),
            "one_thread": {"value": float(statistics.median([r[0] for r in one])), "unit": "predictions/s",
                           "min": float(min(r[0] for r in one)), "max": float(max(r[0] for r in one)),
                           "runs": len(one), "sample": f"{one[0][1]} C5 predictions per run"},
            "oracle_time_to_converge": conv}


def preds_per_iter(nx: int, ny: int) -> int:
    return (2 * (nx // 32) - 1) * (2 * (ny // 32) - 1)


def domain(world: int, scaling: str):
    """strong: the C5 domain on every N; weak: a 1024 x 2048-point block per GPU
    (1024x2048, 2048x2048, 2048x4096, 4096x4096)."""
    if scaling == "strong":
        return NX, NY
    py, px = GRIDS[world]
    return 1024 * px, 2048 * py


def bench_config(T: int, grid, tensor: bool, nx: int = NX, ny: int = NY, scaling: str = "strong") -> dict:
    wl = ("C5: 4097x4097 points, m=32 (65,025 predictions/iteration)" if (nx, ny) == (NX, NY) else
          f"C5 weak scaling: {nx + 1}x{ny + 1} points, m=32 ({preds_per_iter(nx, ny):,} predictions/iteration)")
    return {"workload": wl + f", {T} MFP iterations + final phase per step",
            "nx": nx, "ny": ny, "m": 32, "iters_per_step": T, "grid": list(grid), "scaling": scaling,
            "subsolver": "sdnet d=128 L_h=3 (W-rand)", "gelu": "tanh" if tensor else "erf",
            "l2": "flushed between steps (512 MB write, outside the events)",
            "parallelism": f"domain {grid[0]}x{grid[1]}"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle  # noqa: F401
    times, n_last, thr = [], 0, 1
    for i in range(args.warmup + args.steps):
        rate, n, dt, thr = cpu_oracle_rate(target_s=4.0)
        if i >= args.warmup:
            times.append((n, dt))
        n_last = n
    tot_n = sum(n for n, _ in times)
    tot_t = sum(t for _, t in times)
    v = tot_n / tot_t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "predictions/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot_t / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (GP boundary, W-rand SDNet weights)",
            "config": bench_config(args.iters, GRIDS.get(args.gpus, (1, 1)), args.precision != "fp32",
                                   *domain(args.gpus if args.gpus in GRIDS else 1, args.scaling), args.scaling),
            "cpu_baseline": {"value": v, "unit": "predictions/s", "cores": thr, "kind": "oracle",
                             "sample": f"{n_last} C5 subdomain SDNet predictions per step from the initial "
                                       "lattice (fp64 oracle, exact-erf GELU; a bounded sample of one "
                                       "iteration's work)"},
            "e2e": {"value": v, "unit": "predictions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ boundary IO roofline
IO_N = 16384   # 16385^2 grid: 134 MB line lattice + 134 MB batch, together > 126 MB L2


def boundary_io_bench(mfp, torch, peaks, reps: int = 10, flush_l2: bool = True) -> dict:
    """a1 gather and a6 scatter (+ a8 update-norm reduction) as standalone kernels
    (mfp_gather_phase / mfp_scatter_phase) on a lattice larger than L2, phase 0
    (262,144 subdomains), L2 flushed before every launch (outside the events):
    achieved GB/s of ALGORITHMIC bytes vs the measured HBM copy bandwidth."""
    from mfp_inputs import gp_boundary
    stream = torch.cuda.Stream()
    cfg = mfp.make_config(IO_N, IO_N, precision=mfp.FP32, subsolver=mfp.EXACT_LAPLACE, check_every=16)
    m = mfp.Mfp(cfg, mfp.make_net(), None, stream=stream)
    g = torch.from_numpy(gp_boundary(IO_N, IO_N, 0)).cuda()
    m.solve_device(g, 1, 0.0, None)                  # a real lattice state (one exact iteration)
    B, _ = mfp.mfp_gather_phase(m.ctx, 0, 0)
    gb = torch.empty((B, 128), dtype=torch.float32, device="cuda")
    pred = torch.randn((B, 61), dtype=torch.float32, device="cuda")
    flush = torch.zeros(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    flush_sink = torch.zeros((), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()

    def timed(fn):
        ms = 0.0
        for i in range(reps + 2):
            if flush_l2:
                # evict the lattice by READING a buffer larger than L2: the lines
                # left behind are clean (a write-flush would leave ~126 MB of
                # dirty lines whose write-back the timed kernel would pay for)
                with torch.cuda.stream(stream):
                    flush_sink.copy_(flush.amax())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            if i >= 2:
                ms += e0.elapsed_time(e1)
        return ms / reps

    ms_g = timed(lambda: mfp.mfp_gather_phase(m.ctx, 0, 0, gb, B))
    ms_s = timed(lambda: mfp.mfp_scatter_phase(m.ctx, 0, 0, pred, B, want_norm=False))
    hbm = peaks.get("hbm_gbs", 6650.0)
    gbytes, sbytes = 128 * 4 * 2, 61 * 4 * 2 + 62 * 4   # per subdomain
    out = {"workload": f"{IO_N + 1}^2 grid, phase 0 = {B} subdomains; lattice "
                       f"{m.lines_bytes() / 1e6:.0f} MB (> L2), L2 flushed before each launch by reading a "
                       "512 MB buffer (clean lines; outside the events)",
           "peak_gbs": hbm, "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback",
           "gather": {"kernel": "k_gather_phase (a1)", "us": 1000 * ms_g, "bytes_per_subdomain": gbytes,
                      "note": "512 B perimeter read + 512 B batch write",
                      "gbs": B * gbytes / (ms_g / 1000) / 1e9},
           "scatter": {"kernel": "k_scatter_phase (a6 + the a8 reduction, last block)", "us": 1000 * ms_s,
                       "bytes_per_subdomain": sbytes,
                       "note": "244 B predictions + 244 B old values read, 248 B written (centre twice)",
                       "gbs": B * sbytes / (ms_s / 1000) / 1e9}}
    for k in ("gather", "scatter"):
        out[k]["frac"] = out[k]["gbs"] / hbm
    m.close()
    del flush
    return out


def sdnet_batch_sweep(m, torch, stream, sizes=(1024, 2048, 4096, 8192, 16384, 32768, 65536), reps: int = 5):
    """C3 row of BASELINE.json: batched SDNet inference throughput (mfp_sdnet_batch,
    61 centre-line queries) over batch sizes; N(0,1) boundary vectors."""
    from mfp_inputs import random_boundaries
    out = []
    for B in sizes:
        gb = torch.from_numpy(random_boundaries(B, seed=7)).cuda()
        y = torch.empty((B, 61), dtype=torch.float32, device="cuda")
        torch.cuda.synchronize()
        m.sdnet_batch(gb, out=y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(m.stream)
        for _ in range(reps):
            m.sdnet_batch(gb, out=y)
        e1.record(m.stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out.append({"batch": B, "ms": ms, "predictions_per_s": B / (ms / 1000.0)})
    return out


def halo_line(rep, prof, world: int) -> dict:
    """a7 against the NVLink roofline (north_star): bytes this rank sends per
    exchange over the side-stream span of transport + unpack (CUDA events in
    mfp_profile_iterations), vs the measured 770 GB/s per-direction peer copy of
    B200_PROFILING.md.  Latency-bound by design: tens of KB per exchange."""
    b = rep.halo_bytes_sent / max(rep.iterations, 1)
    out = {"bytes_per_iter_rank0": b, "msgs_per_iter": rep.halo_msgs_per_iter}
    if world > 1 and prof.ms_halo > 0:
        gbs = b / (prof.ms_halo / 1000.0) / 1e9
        out.update({"us_per_exchange": 1000.0 * prof.ms_halo, "gbs": gbs, "peak_gbs": 770.0,
                    "frac": gbs / 770.0, "peak_source": "B200_PROFILING.md measured peer copy, per direction"})
    return out


def nccl_summary(path):
    """Transport lines of rank 0's NCCL INFO log (P2P / NVLS / SHM / NET)."""
    if not path or not os.path.exists(path):
        return None
    kinds = {}
    nvls = False
    for line in open(path, errors="replace"):
        if " via " in line:
            k = line.split(" via ", 1)[1].split()[0]
            kinds[k] = kinds.get(k, 0) + 1
        if "NVLS" in line:
            nvls = True
    return {"log": os.path.relpath(path, ROOT), "channels_via": kinds, "nvls_mentioned": nvls}


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_2308_14258_b200 as mfp
    from mfp_inputs import gp_boundary, random_weights

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE {world}"
    assert world in GRIDS, "supported GPU counts: 1, 2, 4, 8"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    nccl_log = None
    if world > 1:
        # NCCL's INFO log (which transport / NVLS each channel uses) to a file, not
        # stdout: the evidence that the halo really crossed NVLink is kept
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        nccl_log = os.path.join(ROOT, "gpurun_out", f"nccl_debug_rank{rank}.log")
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", nccl_log)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
        obj = [mfp.mfp_nccl_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = mfp.mfp_nccl_comm_init(world, obj[0], rank)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    grid = GRIDS[world]
    nx, ny = domain(world, args.scaling)
    ppi = preds_per_iter(nx, ny)
    prec = {"bf16": mfp.BF16, "fp16": mfp.FP16, "fp32": mfp.FP32}[args.precision]
    tensor = prec != mfp.FP32
    cfg = mfp.make_config(nx, ny, grid, precision=prec, subsolver=mfp.SDNET, check_every=16)
    net = mfp.make_net(gelu=1 if tensor else 0)
    w = random_weights(0)
    stream = torch.cuda.Stream(device=dev)
    m = mfp.Mfp(cfg, net, w, rank=rank, nccl_comm=comm, stream=stream)
    if world > 1 and args.halo in ("p2p", "put"):
        handles = [None] * world
        dist.all_gather_object(handles, mfp.mfp_p2p_export(m.ctx))
        mfp.mfp_p2p_open(m.ctx, handles)
        if args.halo == "put":
            mfp.mfp_p2p_set_mode(m.ctx, mfp.P2P_PUT)
        barrier()
    g_host = gp_boundary(nx, ny, 0)
    g_dev = torch.from_numpy(g_host).to(dev)
    u_dev = torch.empty((ny + 1, nx + 1), dtype=torch.float32, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    T = args.iters

    def step_device():
        return m.solve_device(g_dev, T, 0.0, u_dev)

    # warm-up
    for _ in range(args.warmup):
        rep = step_device()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches = 0
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(float(i))                     # L2 flush, outside the events
                ev[i][0].record(stream)
            rep = step_device()
            launches += rep.gpu_launches
            with torch.cuda.stream(stream):
                ev[i][1].record(stream)
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    ms = max_over_ranks(ms)
    preds = ppi * T * args.steps
    value = preds / (ms / 1000.0)

    # self-check of the distributed run: rank 0 re-solves the same grid with every
    # rank emulated on its own GPU (MFP_ALL_RANKS: same plans, kernels and per-rank
    # batches; device copies instead of NCCL) and compares the final fields
    parity = None
    if world > 1:
        if rank == 0:
            me = mfp.Mfp(cfg, net, w, rank=mfp.ALL_RANKS, stream=stream)
            u_e = torch.empty_like(u_dev)
            me.solve_device(g_dev, T, 0.0, u_e)
            torch.cuda.synchronize()
            diff = float((u_e - u_dev).abs().max())
            parity = {"vs": "MFP_ALL_RANKS emulation of the same grid on rank 0's GPU, same T",
                      "max_abs_diff": diff, "bit_identical": bool(torch.equal(u_e, u_dev)),
                      "max_abs_u": float(u_dev.abs().max())}
            me.close()
            del u_e
        barrier()

    # e2e through the public host API: H2D of g + D2H of u inside the timed
    # region, from / into pinned host buffers
    if args.no_extras:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": ppi * T * args.steps / (ms / 1000.0),
                              "unit": "predictions/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                              "ms_per_step": ms / args.steps, "note": "--no-extras (launch-list run)"}), flush=True)
        m.close()
        if comm is not None:
            mfp.mfp_nccl_comm_destroy(comm)
        if world > 1:
            dist.destroy_process_group()
        return
    u_pin = torch.empty((ny + 1, nx + 1) if rank == 0 else (1, 1), dtype=torch.float32).pin_memory()
    g_pin = torch.from_numpy(g_host).pin_memory()
    u_host, g_host = u_pin.numpy(), g_pin.numpy()
    for _ in range(1):
        mfp.mfp_solve(m.ctx, g_host, T, 0.0, u_host)
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        mfp.mfp_solve(m.ctx, g_host, T, 0.0, u_host)
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    barrier()
    e2e = {"value": preds / e2e_s, "unit": "predictions/s", "h2d_bytes_per_step": g_host.nbytes,
           "d2h_bytes_per_step": (nx + 1) * (ny + 1) * 4 if rank == 0 else 0}

    # roofline of the dominant kernel (the tcgen05 chain), events on its stream
    prof = m.profile(8)
    chain_ms = prof.chain_ms_total / max(prof.chain_launches, 1)
    flop_per_launch = prof.chain_rows / max(prof.chain_launches, 1) * HIDDEN_FLOP_PER_ROW
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    # fp16 and bf16 dense tensor rates are equal (guide: 2.25 PF each), so the
    # measured bf16 cuBLAS peak is the denominator for both; fp32 SIMT peak is
    # derived: 148 SMs x 128 lanes x 2 FLOP x 1.965 GHz = 74.4 TFLOP/s.
    peak = peaks.get("bf16_tflops_sustained", 1400.0) if tensor else 74.4
    achieved = flop_per_launch / (chain_ms / 1000.0) / 1e12
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(tfile):
        traffic = json.load(open(tfile)).get("chain_tc_dram_bytes_per_launch")
    burst = peaks.get("bf16_tflops", 1630.0)
    roofline = {"bound": "tensor" if tensor else "alu", "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                # both measured peaks are reported: the sustained one (a kernel timed inside
                # a long step) and the burst one (the stricter denominator)
                "frac_vs_burst_peak": achieved / burst if tensor else None,
                "burst_peak": burst if tensor else None,
                "kernel": "k_chain_tc2 (hidden GEMM chain a4 + epilogues a3/a5/a6)" if tensor else "k_chain_fp32",
                "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (kernel timed inside a long step)"
                if tensor else "derived fp32 SIMT peak (DESIGN.md §7)",
                "chain_ms_per_launch": chain_ms, "chain_share_of_iteration":
                    prof.chain_ms_total / (prof.ms_per_iter * prof.iterations),
                "iteration_breakdown_ms": {
                    "iteration": prof.ms_per_iter, "chain_per_phase": prof.ms_chain,
                    "gather_embed_per_phase": prof.ms_gather_embed, "halo": prof.ms_halo,
                    "delta_per_check": prof.ms_delta,
                    "note": "mfp_profile_iterations: CUDA events around every kernel (no graphs), "
                            "so the iteration here includes launch gaps the graph-replayed solve avoids"}}
    if tensor:
        # what actually bounds the d = 128 chain: one MUFU tanh per GELU,
        # (n_hidden + 1) x d GELUs per row, against 16 MUFU lanes / clk / SM (tools/ubench)
        # x the SMs x the maximum SM clock (nominal; the chain's own clock under this
        # load is lower)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        clk_mhz = (clk.summary().get("sm_max_mhz") or 1965)
        gelus = prof.chain_rows / max(prof.chain_launches, 1) * 4 * 128
        sfu_peak = 16 * sms * clk_mhz * 1e6 / 1e9
        sfu_ach = gelus / (chain_ms / 1000.0) / 1e9
        roofline["sfu_view"] = {"bound": "alu", "unit": "G GELU/s", "achieved": sfu_ach, "peak": sfu_peak,
                                "frac": sfu_ach / sfu_peak, "gelus_per_launch": gelus,
                                "peak_source": f"16 MUFU.TANH lanes/clk/SM (tools/ubench) x {sms} SMs x "
                                               f"{clk_mhz} MHz (max SM clock)"}

    # time-to-converge (SDNet bf16, tol 1e-3 max|g|, c = 16)
    ttc = None
    if not args.no_converge:
        tol = 1e-3 * float(np.max(np.abs(g_host)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        with torch.cuda.stream(stream):
            e0.record(stream)
        rc = m.solve_device(g_dev, 20000, tol, u_dev)
        with torch.cuda.stream(stream):
            e1.record(stream)
        torch.cuda.synchronize()
        ttc = {"ms": max_over_ranks(e0.elapsed_time(e1)), "iterations": rc.iterations,
               "ms_without_final_phase": max_over_ranks(rc.ms_total - rc.ms_final),
               "converged": bool(rc.converged), "tol": tol, "last_delta": rc.last_delta,
               "note": "W-rand SDNet weights: the fixed point is not physically meaningful (SURVEY exp-5)"}
        # the same MFP with the exact discrete-Laplace subsolver: a provable fixed
        # point (the global 5-point solution), so time-to-converge is meaningful
        cfg_x = mfp.make_config(nx, ny, grid, precision=mfp.FP32, subsolver=mfp.EXACT_LAPLACE, check_every=16)
        mx = mfp.Mfp(cfg_x, net, None, rank=rank, nccl_comm=comm, stream=stream)
        tol_x = 1e-6 * float(np.max(np.abs(g_host)))
        barrier()
        with torch.cuda.stream(stream):
            e0.record(stream)
        rx = mx.solve_device(g_dev, 200000, tol_x, u_dev)
        with torch.cuda.stream(stream):
            e1.record(stream)
        torch.cuda.synchronize()
        ttc_x = {"ms": max_over_ranks(e0.elapsed_time(e1)), "iterations": rx.iterations,
                 "ms_without_final_phase": max_over_ranks(rx.ms_total - rx.ms_final),
                 "converged": bool(rx.converged), "tol": tol_x, "last_delta": rx.last_delta,
                 "subsolver": "exact discrete-Laplace (fp32)"}
        if rank == 0:
            try:
                sys.path.insert(0, os.path.join(ROOT, "tests"))
                from _refsolve import dst_laplace
                ref = dst_laplace(nx, ny, g_host.astype(np.float64))
                ttc_x["max_err_vs_discrete_solution"] = float(np.max(np.abs(u_dev.cpu().numpy() - ref)))
                ttc_x["mae_vs_discrete_solution"] = float(np.mean(np.abs(u_dev.cpu().numpy() - ref)))
            except Exception as e:  # noqa: BLE001
                ttc_x["err_check"] = f"skipped: {e}"
        ttc = {"sdnet_w_rand": ttc, "exact_subsolver": ttc_x}
        mx.close()
        # the paper's stop rule: MAE < 0.05 vs the discrete solution, with
        # the SDNet weights fitted on the boundaries the MFP iteration produces and
        # through the chain's bf16 operand rounding (weights/sdnet_fit_d128_mfp.npy,
        # DESIGN.md §9), bf16 operands, on the paper's strong-scaling domain (2049^2,
        # P:179) and on the bench domain
        # (precision-specific: the fit trains through its own operand rounding)
        fit_prec = mfp.FP16 if prec == mfp.FP16 else mfp.BF16
        wfit = os.path.join(ROOT, "weights", "sdnet_fit_d128_mfp_fp16.npy" if fit_prec == mfp.FP16
                            else "sdnet_fit_d128_mfp.npy")
        if os.path.exists(wfit) and tensor:
            w_fit = np.load(wfit)
            for name, (fx, fy) in (("paper_2049", (2048, 2048)), ("bench_domain", (nx, ny))):
                gf = g_host if (fx, fy) == (nx, ny) else gp_boundary(fx, fy, 0)
                ref_f = None
                flag = torch.zeros(1, device=dev)
                if rank == 0:
                    sys.path.insert(0, os.path.join(ROOT, "tests"))
                    from _refsolve import dst_laplace
                    ref_f = torch.from_numpy(dst_laplace(fx, fy, gf.astype(np.float64)).astype(np.float32)).to(dev)
                cfg_f = mfp.make_config(fx, fy, grid, precision=fit_prec, subsolver=mfp.SDNET, check_every=16)
                mf = mfp.Mfp(cfg_f, mfp.make_net(gelu=1), w_fit, rank=rank, nccl_comm=comm, stream=stream)
                u_f = torch.empty((fy + 1, fx + 1), dtype=torch.float32, device=dev)
                g_arg = torch.from_numpy(gf).to(dev)
                chunk, done, dev_ms, mae, reached = 64, 0, 0.0, float("nan"), False
                while done < 20032:
                    barrier()
                    with torch.cuda.stream(stream):
                        e0.record(stream)
                    mf.solve_device(g_arg, chunk, 0.0, u_f)
                    with torch.cuda.stream(stream):
                        e1.record(stream)
                    torch.cuda.synchronize()
                    dev_ms += max_over_ranks(e0.elapsed_time(e1))
                    done += chunk
                    g_arg = None   # resume from the current lattice
                    flag.zero_()
                    if rank == 0:
                        mae = float((u_f - ref_f).abs().mean())
                        flag[0] = 1.0 if mae < 0.05 else 0.0
                    if world > 1:
                        dist.broadcast(flag, 0)
                    if float(flag[0]) > 0:
                        reached = True
                        break
                ttc[f"sdnet_w_fit_mae_0.05_{name}"] = {
                    "domain": f"{fx + 1}x{fy + 1}", "precision": "fp16" if fit_prec == mfp.FP16 else "bf16",
                    "weights": os.path.basename(wfit), "iterations": done, "reached": reached,
                    "mae": mae, "ms": dev_ms,
                    "note": f"device time of {done // chunk} resumed solves of {chunk} iterations, each including "
                            "the final phase (the MAE needs the field); stop rule of P:179 (paper: 3,200 "
                            "iterations at 2049^2 on 1 A30, 880 s)"}
                mf.close()

    bio = sweep = wide = acc = None
    if tensor:   # every N: the scaling run carries the d = 256 curve
        wide = wide_leg(mfp, torch, stream, cfg, g_dev, u_dev, flush, ppi, peaks, rank=rank, comm=comm,
                        max_over_ranks=max_over_ranks, barrier=barrier)
    if world == 1 and tensor:
        # the tensor-core accuracy mode (split fp16 activations + accurate GELU;
        # holds 3e-3 per field with trained weights, tests/test_gpu_fp16x.py): its
        # throughput cost on the same workload
        cfg_x = mfp.make_config(nx, ny, grid, precision=mfp.FP16X, subsolver=mfp.SDNET, check_every=16)
        acc = wide_leg(mfp, torch, stream, cfg_x, g_dev, u_dev, flush, ppi, peaks, D=128, gelu=2,
                       kernel="k_chain_tc2s (MFP_FP16X: split fp16 activations, d = 128)")
        acc["chain_time_vs_headline_chain"] = acc["roofline"]["chain_ms_per_launch"] / roofline["chain_ms_per_launch"]
        acc["note"] = ("value counts the same 65,025 unique predictions per iteration; each solve of T = 16 "
                       "iterations includes the final phase, so compare chain_time_vs_headline_chain, not value, "
                       "with the headline")
    if world == 1:
        sweep = sdnet_batch_sweep(m, torch, stream)
        bio = boundary_io_bench(mfp, torch, peaks)
    cpu = None
    if rank == 0 and world == 1:
        cpu = cpu_baseline_leg()
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "predictions/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
                "config": bench_config(T, grid, tensor, nx, ny, args.scaling),
                "points_iter_per_s": (nx + 1) * (ny + 1) * T * args.steps / (ms / 1000.0),
                "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "roofline_d256": wide,
                "accuracy_mode_fp16x": acc,
                "cpu_baseline": cpu,
                "time_to_converge": ttc, "sdnet_batch_sweep": sweep, "boundary_io": bio,
                "paper_context": {"note": "the paper's own numbers, other hardware (context, not a baseline; "
                                          "BASELINE.md)",
                                  "mfp_2049_time_to_mae_0.05_s": 880.0, "mfp_2049_iterations_to_mae_0.05": 3200,
                                  "hardware": "1 x A30, mpi4py (P:179, P:187)",
                                  "derived_predictions_per_s": 58.7e3}, "clocks": clk.summary(),
                "halo": halo_line(rep, prof, world), "parity_vs_emulation": parity,
                "nccl_transport": nccl_summary(nccl_log)}
        print(json.dumps(line), flush=True)
    m.close()
    if comm is not None:
        mfp.mfp_nccl_comm_destroy(comm)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
