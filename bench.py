#!/usr/bin/env python
"""bench.py — type-4/5 NFFT throughput on B200 (BASELINE.json metric).

Workload (default, BASELINE.json configs[3] = "C4"): one shared jittered node
set, P = 2^16 nodes (t_p = (p + U[-0.3, 0.3]) / P), complex128 CN(0,1) data,
oversampling eta = 2, the reference's default attenuation mu = 1e-15
(cli.py:62,97), window m = 14.  A STEP = one refined type-5 solve AND one
refined type-4 solve (refine_passes = 1, the path that meets the 1e-10 parity
gate) of B = 1024 signals per GPU.  Unit = nonuniform points through one
solve: each step processes 2 * B * P points per GPU.  Multi-GPU: signals are
sharded by rank (weak scaling: B signals per GPU), each rank builds the
deterministic plan locally, no collective on the data path.

Our arm prints one JSON line with `value` (device-resident inputs, CUDA
events, max over ranks), `e2e` (public API with pinned HOST buffers, copies
inside the timed region), `roofline` (dominant kernel, live per-launch
events), `cpu_baseline` (oracle port on this host's cores, bounded sample),
`clocks` (NVML during the timed region) and `gpu_launches`.

`--impl reference` times the reference algorithm's CPU implementation (the
oracle port, oracle/nfft_oracle.py — the reference is pure Python/numpy, so
its restatement runs at the reference's speed) on all host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "type-4/5 NFFT nonuniform points/s (fp64) at 1/2/4/8 B200; % of HBM roofline"

CONFIGS = {
    # name: P, B (signals per GPU), jitter J, seed
    "c4": dict(P=1 << 16, B=1024, J=0.3, seed=16044, label="C4: batched P=2^16 x 1024 signals, one node set"),
    "c2": dict(P=4096, B=64, J=0.3, seed=16042, label="C2: batched P=4096 x 64 signals"),
    "c3": dict(P=1 << 20, B=1, J=0.4, seed=16043, label="C3: single transform P=2^20"),
    "c1": dict(P=64, B=1, J=0.3, seed=16041, label="C1: single transform P=64"),
}
ETA = 2
MU = 1e-15
PASSES = 1

# Algorithmic HBM bytes per nonuniform point: spread 48,
# gather 48, FFT over the 2P grid 64, FFT over a P vector 32 (elementwise
# work 0).  One refined (passes=1) type-5 or type-4 solve = 464 B/pt.  The
# fused kernels each implement parts of that budget; per step (one refined
# type-5 + one refined type-4) the launches of each kernel carry:
ALGO_BYTES_PER_POINT_STEP = {
    "spread": 3 * 48,            # 3 spreads (spread_p; spread_b for other layouts)
    "gather": 3 * 48,            # 3 gathers (gather_p; gather_b = its fallback for wide node blocks)
    "chain_col": 3 * 32 + 16,    # 3 x (FFT_2P column pass) + 1 x (IFFT_P column pass)
    "chain_band": 3 * 48,        # 3 x (FFT_2P row pass + IFFT_P column pass)
    "chain_mid": 4 * 32,         # 4 x (IFFT_P row pass + FFT_P column pass)
    "chain_pad": 3 * 48,         # 3 x (FFT_P row pass + IFFT_2P column pass)
    "chain_row": 3 * 32 + 16,    # 3 x (IFFT_2P row pass) + 1 x (FFT_P row pass)
    # batch-minor chains (batches >= 16): same stages, plus the two layout-boundary kernels
    # (only one of the chain_* / bm_* families runs for a given batch)
    "bm_col": 3 * 32,            # 3 x FFT_2P column pass
    "bm_colin": 16,              # 1 x IFFT_P column pass (type-4 input, signal-major -> batch-minor)
    "bm_band": 3 * 48,
    "bm_mid": 4 * 32,
    "bm_pad": 3 * 48,
    "bm_row": 3 * 32,            # 3 x IFFT_2P row pass
    "bm_rowout": 16,             # 1 x FFT_P row pass (type-5 output, batch-minor -> signal-major)
    # one-CTA fused small solves (P <= 256): a whole refined solve per launch, so only the
    # operand read and the result write reach HBM (2 launches per step: type-5, type-4)
    "tiny": 2 * 32,
}


def make_nodes(P: int, J: float, seed: int):
    """Nodes t_p = ((p + u_p)/P) mod 1, u ~ U[-J, J] (Philox key = seed), as the oracle's make_inputs."""
    import numpy as np

    rng = np.random.Generator(np.random.Philox(key=seed))
    u = rng.uniform(-J, J, P)
    t = np.mod((np.arange(P) + u) / P, 1.0)
    t[t >= 1.0] = 0.0
    return t


# ------------------------------------------------------------------ clocks

_REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks", 0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x10: "sync_boost",
    0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake", 0x100: "display_clocks",
}


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons while the timed region runs."""

    def __init__(self, dev: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in _REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------- CPU baseline

_W = {}


def _cpu_init(t, a, eta):
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import nfft_oracle as O

    _W["O"] = O
    _W["plan"] = O.Plan.build(t, a, eta)
    _W["t"] = t


def _cpu_solve(seed):
    import numpy as np

    O = _W["O"]
    P = _W["t"].size
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal(P) + 1j * rng.standard_normal(P)) / math.sqrt(2.0)
    O.refine5(_W["plan"], x, PASSES)
    O.refine4(_W["plan"], x, PASSES)
    return 2 * P


class CpuReference:
    """The reference algorithm (oracle port) on `cores` host processes, plan built once per worker."""

    def __init__(self, cfg, a):
        import multiprocessing as mp

        self.cores = max(1, os.cpu_count() or 1)
        t = make_nodes(cfg["P"], cfg["J"], cfg["seed"])
        self.pool = mp.get_context("fork").Pool(self.cores, initializer=_cpu_init, initargs=(t, a, ETA))
        self.P = cfg["P"]
        # signals per sample: one per core (each worker: one refined type-5 + one refined type-4)
        self.nsig = min(self.cores, max(1, cfg["B"] * 4))
        self._seed = 0

    def step(self):
        seeds = list(range(self._seed, self._seed + self.nsig))
        self._seed += self.nsig
        t0 = time.perf_counter()
        pts = sum(self.pool.map(_cpu_solve, seeds, chunksize=1))
        return pts, time.perf_counter() - t0

    def close(self):
        self.pool.close()
        self.pool.join()

    def describe(self):
        return (f"{self.nsig} signals x P={self.P}, refined type-5 + type-4 (passes={PASSES}) per signal, "
                f"plan prebuilt per worker, {self.cores} processes, oracle/nfft_oracle.py (numpy "
                f"restatement of the reference)")


# ------------------------------------------------------------------- main


def dist_setup():
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(local)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_reference(args, cfg):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import nfft_oracle as O

    a = O.damping(MU, cfg["P"], ETA)
    ref = CpuReference(cfg, a)
    for _ in range(args.warmup):
        ref.step()
    pts = 0
    secs = 0.0
    for _ in range(args.steps):
        p, s = ref.step()
        pts += p
        secs += s
    ref.close()
    v = pts / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["label"], "P": cfg["P"], "eta": ETA, "mu": MU, "refine_passes": PASSES,
                   "spread_width": 14},
        "cpu_baseline": {"value": v, "unit": "points/s", "cores": ref.cores, "kind": "port",
                         "sample": ref.describe()},
        "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=0, help="cap on timed e2e steps (0: all K steps)")
    ap.add_argument("--batch", type=int, default=0, help="override signals per GPU (experiments)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", type=int, default=0, choices=[0, 1, 2],
                    help="run the step's type-5 and type-4 solves on 1 or 2 CUDA streams (0: 2 for the "
                         "small configs C1-C3, whose latency-bound solves overlap, else 1)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    cfg = dict(CONFIGS[args.config])
    if args.streams == 0:
        # mid-size latency-bound configs (C3) overlap their two solves on two streams;
        # the one-CTA small solves (C1) and C2 are host-bound, where the extra stream
        # handling costs more than the overlap gains (C1: 0.058 vs 0.075 ms/step)
        pts = (args.batch or cfg["B"]) * cfg["P"]
        args.streams = 2 if (1 << 18) < pts <= (1 << 22) else 1
    if args.batch:
        cfg["B"] = args.batch
        cfg["label"] += f" (batch override {args.batch})"
    if args.impl == "reference":
        return run_reference(args, cfg)

    import numpy as np
    import torch

    import paper_1604_06236_b200 as nf
    from paper_1604_06236_b200 import _lib

    world, rank, local = dist_setup()
    dev = local
    P, B = cfg["P"], cfg["B"]

    # ---- plan (once per node set; deterministic, built locally on every rank)
    t = make_nodes(P, cfg["J"], cfg["seed"])
    grid = nf.validate_grid(t)
    params = nf.MethodParams.from_mu(MU, P, ETA)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = nf.build_plan(grid, params, device=dev)
    torch.cuda.synchronize()
    plan_ms = 1e3 * (time.perf_counter() - t0)
    # warm rebuild of the same node set (the first build also pays the
    # library's one-time costs: lazy module loading, FFT twiddle tables)
    grid2 = nf.validate_grid(t)
    grid2.device_handle(dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    nf.build_plan(grid2, params, device=dev)
    torch.cuda.synchronize()
    plan_warm_ms = 1e3 * (time.perf_counter() - t0)
    del grid2

    # ---- device-resident inputs (this rank's shard of signals), seeded
    gen = torch.Generator(device=f"cuda:{dev}")
    gen.manual_seed(cfg["seed"] * 1000 + rank)
    s_in = torch.complex(torch.randn(B, P, generator=gen, device=f"cuda:{dev}", dtype=torch.float64),
                         torch.randn(B, P, generator=gen, device=f"cuda:{dev}", dtype=torch.float64)) / math.sqrt(2)
    A_in = torch.complex(torch.randn(B, P, generator=gen, device=f"cuda:{dev}", dtype=torch.float64),
                         torch.randn(B, P, generator=gen, device=f"cuda:{dev}", dtype=torch.float64)) / math.sqrt(2)
    out5 = torch.empty_like(s_in)
    out4 = torch.empty_like(A_in)
    stream = torch.cuda.current_stream(dev)
    side = torch.cuda.Stream(dev)  # the type-4 solve of a step runs beside the type-5 solve

    def step():
        if args.streams == 2:
            side.wait_stream(stream)
            nf.refine_type5(plan, s_in, passes=PASSES, out=out5)
            with torch.cuda.stream(side):
                nf.refine_type4(plan, A_in, passes=PASSES, out=out4)
            stream.wait_stream(side)
        else:
            nf.refine_type5(plan, s_in, passes=PASSES, out=out5)
            nf.refine_type4(plan, A_in, passes=PASSES, out=out4)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _lib.load().nfft45_launch_count()
    # small solves replay cached CUDA graphs (library: P * batch <= 2^22, passes <= 1);
    # per-launch profiling would switch that off, so they are profiled in a second pass
    graphed = P * B <= (1 << 22) and PASSES <= 1
    _lib.profile_enable(not graphed)
    with ClockSampler(dev) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    _lib.profile_enable(False)
    launches = _lib.load().nfft45_launch_count() - l0
    kprof = _lib.profile_read()
    kernel_timing = "live CUDA events around every launch of the timed region"
    if graphed:
        # small configs replay cached CUDA graphs, whose kernels the per-launch
        # events cannot see: time the same K steps once more with the graphs off
        # (the library bypasses its graph cache while profiling), one stream
        _lib.profile_enable(True)
        for _ in range(args.steps):
            nf.refine_type5(plan, s_in, passes=PASSES, out=out5)
            nf.refine_type4(plan, A_in, passes=PASSES, out=out4)
        torch.cuda.synchronize()
        _lib.profile_enable(False)
        kprof = _lib.profile_read()
        kernel_timing = ("live CUDA events around every launch of a second, un-graphed pass of the same "
                         "K steps on one stream (the timed region replays CUDA graphs)")
    kernels_raw = dict(kprof)
    fam = {}  # spread_p/spread_b -> spread, gather_p/gather_b -> gather
    for name, (cnt, kms) in kprof.items():
        key = name.split("_")[0] if name.split("_")[0] in ("spread", "gather") else name
        c0, m0 = fam.get(key, (0, 0.0))
        fam[key] = (max(c0, cnt), m0 + kms)
    kprof = fam
    barrier(world)
    ms = max_over_ranks(ev0.elapsed_time(ev1), world)
    pts_per_step = 2 * B * P * world
    value = pts_per_step * args.steps / (ms / 1e3)

    # ---- parity spot check on the bench data: forward residual of a few signals
    k = min(B, 4)
    r5 = nf.nfft_type2(out5[:k], grid, device=dev) - s_in[:k]
    r4 = nf.nfft_type1(grid, out4[:k], P, device=dev) - A_in[:k]
    resid5 = float((torch.linalg.norm(r5) / torch.linalg.norm(s_in[:k])).item())
    resid4 = float((torch.linalg.norm(r4) / torch.linalg.norm(A_in[:k])).item())

    # ---- e2e through the public API with pinned host buffers
    del r5, r4
    hs = s_in.cpu().pin_memory()
    hA = A_in.cpu().pin_memory()
    ho5 = torch.empty_like(hs).pin_memory()
    ho4 = torch.empty_like(hA).pin_memory()
    def e2e_step():
        # non_blocking (torch copy_ semantics): the type-4 uploads start while the
        # type-5 downloads drain (and, on two streams, run beside the type-5
        # solve); the synchronize after the loop completes every copy
        if args.streams == 2:
            side.wait_stream(stream)
            nf.refine_type5(plan, hs, passes=PASSES, out=ho5, non_blocking=True)
            with torch.cuda.stream(side):
                nf.refine_type4(plan, hA, passes=PASSES, out=ho4, non_blocking=True)
            stream.wait_stream(side)
        else:
            nf.refine_type5(plan, hs, passes=PASSES, out=ho5, non_blocking=True)
            nf.refine_type4(plan, hA, passes=PASSES, out=ho4, non_blocking=True)

    # warm the host path (graph capture of small solves happens on the second
    # call) until two consecutive steps agree: on a freshly provisioned box the
    # first pinned-memory transfers run several times slower than steady state
    # (a first call on one box ran ~6x slow for its first seconds): at least 3 s
    # and 3 steps of warm-up, then until two consecutive steps agree within 10 %
    warm_ms = []
    wt0 = time.perf_counter()
    for i in range(200):
        w0 = time.perf_counter()
        e2e_step()
        torch.cuda.synchronize()
        warm_ms.append(1e3 * (time.perf_counter() - w0))
        if (i >= 2 and time.perf_counter() - wt0 >= 3.0
                and abs(warm_ms[-1] - warm_ms[-2]) <= 0.1 * warm_ms[-2]):
            break
    barrier(world)
    # the same K steps as the device-resident timing (--e2e-steps caps it for quick runs)
    e2e_steps = max(1, min(args.e2e_steps, args.steps)) if args.e2e_steps > 0 else args.steps
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0, world)
    e2e_value = pts_per_step * e2e_steps / e2e_s
    bytes_io = 2 * B * P * 16  # both solves' inputs (and outputs)

    # ---- roofline of the dominant kernel (live per-launch events above)
    peaks_path = os.path.join(REPO, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        peak, peak_src = float(json.load(open(peaks_path))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    top = max(kprof.items(), key=lambda kv: kv[1][1]) if kprof else ("", (0, 0.0))
    tname, (tcount, tms) = top
    step_kernel_ms = sum(v[1] for v in kprof.values())
    algo = None
    if tname in ALGO_BYTES_PER_POINT_STEP and tcount:
        # algorithmic bytes per launch = (bytes/pt/step x points/step) / launches per step
        algo = ALGO_BYTES_PER_POINT_STEP[tname] * B * P * args.steps / tcount
    roof = None
    if algo and tcount:
        avg_ms = tms / tcount
        achieved = algo / (avg_ms / 1e3) / 1e9
        traffic = None
        tfile = os.path.join(REPO, "profiles", f"traffic_{args.config}.json")
        if os.path.exists(tfile):
            tj = json.load(open(tfile))
            traffic = tj.get(tname, next((v for k, v in tj.items() if k.startswith(tname + "_")), None))
        roof = {"kernel": tname, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "algorithmic_bytes_per_launch": algo,
                "avg_launch_ms": avg_ms, "launches": tcount, "share_of_kernel_time": tms / step_kernel_ms,
                "peak_source": peak_src}

    # per kernel family: algorithmic bytes / live time, and, where the
    # committed ncu capture of this config has it, the kernel's MEASURED DRAM bytes
    # per launch / live launch time (how close each kernel runs to the HBM peak on
    # the traffic it actually moves)
    tfile = os.path.join(REPO, "profiles", f"traffic_{args.config}.json")
    tj = json.load(open(tfile)) if os.path.exists(tfile) else {}
    per_kernel_roofline = {}
    for name, (cnt, kms) in kprof.items():
        if name in ALGO_BYTES_PER_POINT_STEP and kms > 0:
            gbs = ALGO_BYTES_PER_POINT_STEP[name] * B * P * args.steps / (kms / 1e3) / 1e9
            per_kernel_roofline[name] = {"achieved_GBps": gbs, "frac": gbs / peak}
            tb = tj.get(name, next((v for k, v in tj.items() if k.startswith(name + "_")), None))
            if tb and cnt:
                dram = tb / (kms / cnt / 1e3) / 1e9
                per_kernel_roofline[name].update({"dram_GBps": dram, "dram_frac": dram / peak})
    total_algo = sum(ALGO_BYTES_PER_POINT_STEP[k] for k in kprof if k in ALGO_BYTES_PER_POINT_STEP) * B * P
    line = {
        "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["label"], "P": P, "signals_per_gpu": B, "global_batch": B * world, "eta": ETA,
                   "mu": MU, "damping_a": params.damping_a, "spread_width": 14, "refine_passes": PASSES,
                   "jitter": cfg["J"], "parallelism": f"signal-sharded x{world}", "streams": args.streams,
                   "l2": f"inputs larger than L2 ({2 * B * P * 16 / 2**30:.2f} GiB per step)" if B * P >= 1 << 22
                   else "inputs fit in L2 (small config)"},
        "roofline": roof,
        "e2e": {"value": e2e_value, "unit": "points/s", "h2d_bytes_per_step": bytes_io, "d2h_bytes_per_step": bytes_io,
                "steps": e2e_steps, "api": "refine_type5/refine_type4 on pinned CPU tensors (out= pinned)",
                "warmup_steps": len(warm_ms), "warmup_ms_first_last": [round(warm_ms[0], 3), round(warm_ms[-1], 3)]},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "plan_ms": plan_ms,
        "plan_warm_ms": plan_warm_ms,
        # single transforms (the plan is not amortised for C1, C3, C5):
        # the same metric with one warm plan build charged to every step
        "with_plan": ({"value": pts_per_step / ((ms / args.steps + plan_warm_ms) / 1e3), "unit": "points/s",
                       "ms_per_step": ms / args.steps + plan_warm_ms} if B == 1 else None),
        "parity": {"forward_residual_type5": resid5, "forward_residual_type4": resid4},
        "kernels_ms_per_step": {k: v[1] / args.steps for k, v in sorted(kernels_raw.items(), key=lambda kv: -kv[1][1])},
        "kernel_roofline": per_kernel_roofline,
        "kernel_timing": kernel_timing,
        "step_roofline": {"algorithmic_bytes_per_step": total_algo,
                          "achieved_GBps": total_algo / (ms / args.steps / 1e3) / 1e9 / world,
                          "frac": total_algo / (ms / args.steps / 1e3) / 1e9 / world / peak},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ref = CpuReference(cfg, params.damping_a)
        ref.step()  # warm the workers
        pts, secs = ref.step()
        ref.close()
        line["cpu_baseline"] = {"value": pts / secs, "unit": "points/s", "cores": ref.cores, "kind": "port",
                                "sample": ref.describe()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
