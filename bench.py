#!/usr/bin/env python
"""bench.py — type-4/5 NFFT throughput on B200 (BASELINE.json metric).

Workload (default, BASELINE.json configs[3] = "C4"): one shared jittered node
set, P = 2^16 nodes (t_p = (p + U[-0.3, 0.3]) / P), complex128 CN(0,1) data,
oversampling eta = 2, the reference's default attenuation mu = 1e-15
(cli.py:62,97), window m = 14.  A STEP = one refined type-5 solve AND one
refined type-4 solve (refine_passes = 1, the path that meets the 1e-10 parity
gate) of the job's 1024 signals.  Unit = nonuniform points through one solve:
each step processes 2 * 1024 * P points in the whole job.

Multi-GPU: one process per GPU.  `--gpus N` under torchrun uses
the launcher's ranks; invoked directly it re-launches itself under
torch.distributed.run with N ranks (and exits non-zero when fewer than N GPUs
are visible).  C4 is STRONG-scaled by default (1024 signals in total, rank r
solves the contiguous block shard_bounds(1024, N, r); `--scaling weak` keeps
1024 signals per GPU).  Each rank builds the deterministic plan locally; no
collective touches the transform.  The final gather of the outputs to rank 0
(NCCL over NVLink) is timed separately (`gather`), device events, max over
ranks.

Our arm prints one JSON line with `value` (device-resident inputs, CUDA
events, un-instrumented, max over ranks), `e2e` (public API with pinned HOST
torch buffers, copies inside the timed region), `e2e_numpy` (the reference's
own convention: numpy arrays in, numpy arrays out), `roofline` (dominant
kernel: live per-launch events of a second, profiled pass of the same K
steps), `cpu_baseline` (the reference itself from baseline/_ref on this host's
cores, bounded sample; the oracle port only if baseline/_ref is absent),
`clocks` (NVML during the timed region) and `gpu_launches`.

`--impl reference` times the reference's own CPU implementation
(baseline/_ref/nufft1d: build_plan once per worker process, then
refine_type5 / refine_type4 per signal) on all host cores, plus a 1-core
serial figure.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
REF_PATH = os.path.join(REPO, "baseline", "_ref")

METRIC = "type-4/5 NFFT nonuniform points/s (fp64) at 1/2/4/8 B200; % of HBM roofline"

CONFIGS = {
    # name: P, B (signals in the job; per GPU under --scaling weak), jitter J, seed
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


def shard_bounds(batch: int, world: int, rank: int):
    """Same contiguous split as paper_1604_06236_b200.distributed.shard_bounds."""
    base, extra = divmod(batch, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


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


# ------------------------------------------------- CPU reference (baseline)
#
# Workers are SPAWNED (fresh interpreters) with the BLAS / OpenMP thread pools
# pinned to one thread in the environment before they import numpy: one
# process per core, each with its own plan (the reference's plans are
# immutable and rebuilt deterministically), signals dealt out one per task —
# the reference's own batch is a serial loop over signals sharing one plan
# (bench.py:183-205).

_SINGLE_THREAD_ENV = {"OMP_NUM_THREADS": "1", "OPENBLAS_NUM_THREADS": "1", "MKL_NUM_THREADS": "1",
                      "NUMEXPR_NUM_THREADS": "1", "VECLIB_MAXIMUM_THREADS": "1"}
_W = {}


def _reference_available() -> bool:
    return os.path.isdir(os.path.join(REF_PATH, "nufft1d"))


def _cpu_init(t, P, kind):
    """Worker: build the plan once (reference: validate_grid -> MethodParams.from_mu -> build_plan)."""
    import numpy as np

    if kind == "reference":
        sys.path.insert(0, REF_PATH)
        import nufft1d as R  # the unmodified reference package (pip --target baseline/_ref)

        params = R.MethodParams.from_mu(MU, P, ETA)
        _W["plan"] = R.build_plan(R.validate_grid(np.asarray(t)), params)
        _W["r5"] = lambda x: R.refine_type5(_W["plan"], x, passes=PASSES)
        _W["r4"] = lambda x: R.refine_type4(_W["plan"], x, passes=PASSES)
    else:  # the oracle port (bitwise the reference on the golden set), only if baseline/_ref is absent
        from oracle import nfft_oracle as O

        plan = O.Plan.build(np.asarray(t), O.damping(MU, P, ETA), ETA)
        _W["r5"] = lambda x: O.refine5(plan, x, PASSES)
        _W["r4"] = lambda x: O.refine4(plan, x, PASSES)
    _W["P"] = P


def _cpu_solve(seed):
    """One signal: refined type-5 and refined type-4 on CN(0,1) data (2P points); returns (points, secs)."""
    import numpy as np

    P = _W["P"]
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal(P) + 1j * rng.standard_normal(P)) / math.sqrt(2.0)
    t0 = time.perf_counter()
    _W["r5"](x)
    _W["r4"](x)
    return 2 * P, time.perf_counter() - t0


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class CpuReference:
    """The reference (baseline/_ref) on `procs` spawned single-threaded processes."""

    def __init__(self, cfg, procs: int | None = None):
        import multiprocessing as mp

        os.environ.update(_SINGLE_THREAD_ENV)  # inherited by the spawned workers before numpy loads
        self.kind = "reference" if _reference_available() else "port"
        try:
            avail = len(os.sched_getaffinity(0))
        except AttributeError:
            avail = os.cpu_count() or 1
        self.host_cpus = os.cpu_count() or 1
        self.cores = max(1, procs or avail)
        self.P = cfg["P"]
        t = make_nodes(cfg["P"], cfg["J"], cfg["seed"])
        t0 = time.perf_counter()
        self.pool = mp.get_context("spawn").Pool(self.cores, initializer=_cpu_init, initargs=(t, self.P, self.kind))
        self.pool.map(_noop, range(self.cores), chunksize=1)  # every worker has imported + built its plan
        self.startup_s = time.perf_counter() - t0
        # signals per step: one per process (bounded sample of the job's signals)
        self.nsig = self.cores
        self._seed = 0

    def step(self):
        seeds = list(range(self._seed, self._seed + self.nsig))
        self._seed += self.nsig
        t0 = time.perf_counter()
        res = self.pool.map(_cpu_solve, seeds, chunksize=1)
        wall = time.perf_counter() - t0
        return sum(p for p, _ in res), wall, sum(s for _, s in res)

    def close(self):
        self.pool.close()
        self.pool.join()

    def describe(self, job_signals: int):
        what = ("baseline/_ref nufft1d (the unmodified reference: build_plan once per process, then "
                "refine_type5 + refine_type4 per signal)" if self.kind == "reference"
                else "oracle/nfft_oracle.py (numpy restatement; baseline/_ref absent)")
        return (f"{self.nsig} of the job's {job_signals} signals per step (one per process), P={self.P}, "
                f"refined type-5 + type-4 (passes={PASSES}) per signal, {self.cores} single-threaded spawned "
                f"processes; {what}")


def _noop(_):
    return 0


def cpu_reference_figures(cfg, steps: int, warmup: int, serial_signals: int = 2):
    """All-core rate (the baseline) and a 1-core serial rate, with host facts."""
    import numpy as np

    ref = CpuReference(cfg)
    for _ in range(warmup):
        ref.step()
    pts = 0
    secs = 0.0
    for _ in range(steps):
        p, w, _ = ref.step()
        pts += p
        secs += w
    ref.close()
    one = CpuReference(cfg, procs=1)
    one.nsig = serial_signals
    one.step()  # warm
    p1, w1, _ = one.step()
    one.close()
    facts = {"cpu_model": _cpu_model(), "host_cpus": ref.host_cpus, "numpy": np.__version__,
             "serial_1core": {"value": p1 / w1, "unit": "points/s", "cores": 1,
                              "sample": f"{serial_signals} signals, P={cfg['P']}, one process"},
             "worker_startup_s": round(ref.startup_s, 2)}
    if ref.kind == "reference":
        sys.path.insert(0, REF_PATH)
        import nufft1d

        facts["reference_version"] = getattr(nufft1d, "__version__", "0.1.0")
    return ref, pts, secs, facts


# ------------------------------------------------------------------- main


def relaunch_under_torchrun(args) -> int:
    """`bench.py --gpus N` without a launcher: re-run under torch.distributed.run with N ranks."""
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus and not args.oversubscribe:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} requested, {have} CUDA devices visible",
                          "n_gpus": args.gpus}), flush=True)
        return 1
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_setup(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.oversubscribe:
            # test mode: every rank on cuda:0 (independent solves, host-side gloo
            # barriers; no kernel waits on another rank)
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            # NCCL's INFO log lets the driver count the communicator's ranks
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(local)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int, dev: int, backend_gloo: bool) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cpu" if backend_gloo else f"cuda:{dev}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return 0
    ref, pts, secs, facts = cpu_reference_figures(cfg, args.steps, args.warmup)
    v = pts / secs
    job = cfg["B"] * (world if args.scaling == "weak" else 1)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": config_block(cfg, world, args, signals_here=job // world if args.scaling == "strong" else cfg["B"],
                               job=job),
        "cpu_baseline": {"value": v, "unit": "points/s", "cores": ref.cores, "kind": ref.kind,
                         "sample": ref.describe(job)},
        "host": facts,
        "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_block(cfg, world, args, signals_here, job, extra=None):
    P = cfg["P"]
    d = {"workload": cfg["label"], "P": P, "global_batch": job, "signals_per_gpu": signals_here, "eta": ETA,
         "mu": MU, "spread_width": 14, "refine_passes": PASSES, "jitter": cfg["J"],
         "parallelism": f"signal-sharded x{world} ({args.scaling} scaling)", "node_seed": cfg["seed"],
         "l2": (f"inputs larger than L2 ({2 * signals_here * P * 16 / 2**30:.2f} GiB per step per GPU)"
                if signals_here * P >= 1 << 22 else "inputs fit in L2 (small config)")}
    if extra:
        d.update(extra)
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's signals are split across the GPUs; weak: every GPU solves them all")
    ap.add_argument("--e2e-steps", type=int, default=0, help="cap on timed e2e steps (0: all K steps)")
    ap.add_argument("--batch", type=int, default=0, help="override the config's signal count (experiments)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-memory legs (quick kernel runs)")
    ap.add_argument("--oversubscribe", action="store_true",
                    help="test mode: all ranks share cuda:0 over a gloo group (no NCCL)")
    ap.add_argument("--streams", type=int, default=0, choices=[0, 1, 2],
                    help="run the step's type-5 and type-4 solves on 1 or 2 CUDA streams (0: 2 for the "
                         "mid-size single transforms, whose latency-bound solves overlap, else 1)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.batch:
        cfg["B"] = args.batch
        cfg["label"] += f" (batch override {args.batch})"
    if args.impl == "reference":
        return run_reference(args, cfg)
    args.warmup = max(args.warmup, 3)
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and world_env == 1:
        return relaunch_under_torchrun(args)
    if world_env > 1 and world_env != args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"WORLD_SIZE={world_env} but --gpus {args.gpus}"}), flush=True)
        return 2

    import numpy as np
    import torch

    import paper_1604_06236_b200 as nf
    from paper_1604_06236_b200 import _lib

    world, rank, local = dist_setup(args)
    gloo = world > 1 and args.oversubscribe
    dev = local
    P = cfg["P"]
    job = cfg["B"] * (world if args.scaling == "weak" else 1)
    lo, hi = (shard_bounds(job, world, rank) if args.scaling == "strong" else (rank * cfg["B"], (rank + 1) * cfg["B"]))
    B = hi - lo  # this rank's signals
    if B <= 0:
        print(json.dumps({"metric": METRIC, "error": f"rank {rank} has no signals ({job} over {world})"}),
              flush=True)
        return 2
    if args.streams == 0:
        # mid-size latency-bound configs (C3) overlap their two solves on two streams;
        # the one-CTA small solves (C1) and C2 are host-bound, where the extra stream
        # handling costs more than the overlap gains (C1: 0.058 vs 0.075 ms/step)
        args.streams = 2 if (1 << 18) < B * P <= (1 << 22) else 1

    # ---- plan (once per node set; deterministic, built locally on every rank)
    t = make_nodes(P, cfg["J"], cfg["seed"])
    grid = nf.validate_grid(t)
    params = nf.MethodParams.from_mu(MU, P, ETA)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = nf.build_plan(grid, params, device=dev)
    torch.cuda.synchronize()
    plan_ms = 1e3 * (time.perf_counter() - t0)
    # warm rebuilds for a fresh node-set handle (the first build also pays the library's
    # one-time costs: lazy module loading, FFT twiddle tables).  The first rebuild still grows
    # the stream-ordered pool (plan 1 is alive, so a second set of tables is allocated); from
    # then on a rebuilt plan reuses the memory of the one it replaces: plan_warm_ms is the
    # median of three such steady-state rebuilds, all four times are reported.
    rebuild_ms = []
    for _ in range(4):
        grid2 = nf.validate_grid(t)
        grid2.device_handle(dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan2 = nf.build_plan(grid2, params, device=dev)
        torch.cuda.synchronize()
        rebuild_ms.append(1e3 * (time.perf_counter() - t0))
        del plan2, grid2
    plan_warm_ms = sorted(rebuild_ms[1:])[1]

    # ---- device-resident inputs: this rank's rows of the job's seeded signals
    # (row r of the job is drawn from the generator keyed (seed, r // 64), so
    # every rank gets the same rows of the same job, whatever the rank count)
    def rows(first, count, salt):
        chunks = []
        for blk in range(first // 64, (first + count + 63) // 64):
            g = torch.Generator(device=f"cuda:{dev}")
            g.manual_seed((cfg["seed"] * 1000 + salt) * 100003 + blk)
            re = torch.randn(64, P, generator=g, device=f"cuda:{dev}", dtype=torch.float64)
            im = torch.randn(64, P, generator=g, device=f"cuda:{dev}", dtype=torch.float64)
            a, b = max(first, blk * 64) - blk * 64, min(first + count, (blk + 1) * 64) - blk * 64
            chunks.append(torch.complex(re[a:b], im[a:b]) / math.sqrt(2))
        return torch.cat(chunks).contiguous()

    s_in = rows(lo, B, 5)
    A_in = rows(lo, B, 4)
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

    # ---- timed region: un-instrumented (no per-launch events), CUDA events on the launching stream
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _lib.load().nfft45_launch_count()
    _lib.profile_enable(False)
    with ClockSampler(dev) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = _lib.load().nfft45_launch_count() - l0
    barrier(world)
    ms = max_over_ranks(ev0.elapsed_time(ev1), world, dev, gloo)
    pts_per_step = 2 * job * P
    value = pts_per_step * args.steps / (ms / 1e3)

    # ---- second pass of the same K steps with per-launch CUDA events (kernel
    # table + roofline); the library bypasses its graph cache while profiling
    _lib.profile_enable(True)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(args.steps):
        nf.refine_type5(plan, s_in, passes=PASSES, out=out5)
        nf.refine_type4(plan, A_in, passes=PASSES, out=out4)
    p1.record(stream)
    torch.cuda.synchronize()
    _lib.profile_enable(False)
    profiled_ms = p0.elapsed_time(p1)
    kprof = _lib.profile_read()
    kernel_timing = ("live CUDA events around every launch of a second, profiled pass of the same K steps "
                     "on one stream (the timed region runs without per-launch events)")
    kernels_raw = dict(kprof)
    fam = {}  # spread_p/spread_b -> spread, gather_p/gather_b -> gather
    for name, (cnt, kms) in kprof.items():
        key = name.split("_")[0] if name.split("_")[0] in ("spread", "gather") else name
        c0, m0 = fam.get(key, (0, 0.0))
        fam[key] = (max(c0, cnt), m0 + kms)
    kprof = fam

    # ---- final gather of the type-5 outputs to rank 0 (the job's only collective), timed alone
    gather = None
    if world > 1:
        import torch.distributed as dist

        from paper_1604_06236_b200.distributed import gather_rows

        src = out5.cpu() if gloo else out5
        barrier(world)
        torch.cuda.synchronize()
        g0 = time.perf_counter()
        ge0, ge1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ge0.record(stream)
        full = gather_rows(src, job, world, rank)
        ge1.record(stream)
        torch.cuda.synchronize()
        gwall = time.perf_counter() - g0
        gms = max_over_ranks(ge0.elapsed_time(ge1) if not gloo else 1e3 * gwall, world, dev, gloo)
        gbytes = 16 * P * (job - B if rank == 0 else 0)
        gbytes = max_over_ranks(float(gbytes), world, dev, gloo)
        ok = None
        if rank == 0:
            ok = bool(full.shape == (job, P)) and bool(torch.equal(full[:B].to(out5.device), out5))
        gather = {"ms": gms, "bytes_into_rank0": gbytes, "GBps": gbytes / (gms / 1e3) / 1e9 if gms > 0 else None,
                  "backend": "gloo (oversubscribed test mode)" if gloo else "nccl",
                  "what": "type-5 outputs of one step, [job, P] complex128 onto rank 0", "rank0_rows_ok": ok,
                  "value_with_gather": pts_per_step / ((ms / args.steps + gms) / 1e3)}
        del full, src
        dist.barrier()

    # ---- parity spot check on the bench data: forward residual of a few signals
    k = min(B, 4)
    r5 = nf.nfft_type2(out5[:k], grid, device=dev) - s_in[:k]
    r4 = nf.nfft_type1(grid, out4[:k], P, device=dev) - A_in[:k]
    resid5 = float((torch.linalg.norm(r5) / torch.linalg.norm(s_in[:k])).item())
    resid4 = float((torch.linalg.norm(r4) / torch.linalg.norm(A_in[:k])).item())
    del r5, r4

    e2e = e2e_np = None
    bytes_io = 2 * B * P * 16  # both solves' inputs (and outputs), this rank
    if not args.no_e2e:
        # ---- e2e through the public API with pinned host torch buffers
        hs = s_in.cpu().pin_memory()
        hA = A_in.cpu().pin_memory()
        ho5 = torch.empty_like(hs).pin_memory()
        ho4 = torch.empty_like(hA).pin_memory()

        def e2e_step():
            # non_blocking (torch copy_ semantics): the type-4 uploads start while the
            # type-5 downloads drain; the synchronize after the loop completes every copy
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
        e2e_steps = max(1, min(args.e2e_steps, args.steps)) if args.e2e_steps > 0 else args.steps
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_s = max_over_ranks(time.perf_counter() - t0, world, dev, gloo)
        e2e = {"value": pts_per_step * e2e_steps / e2e_s, "unit": "points/s", "h2d_bytes_per_step": bytes_io,
               "d2h_bytes_per_step": bytes_io, "steps": e2e_steps,
               "api": "refine_type5/refine_type4 on pinned CPU torch tensors (out= pinned)",
               "warmup_steps": len(warm_ms), "warmup_ms_first_last": [round(warm_ms[0], 3), round(warm_ms[-1], 3)]}
        del ho5, ho4, hA

        # ---- e2e in the reference's own convention: numpy arrays in, numpy arrays out
        # (host_array validation incl. the finiteness scan, pageable memory)
        ns, nA = s_in.cpu().numpy(), A_in.cpu().numpy()
        del hs
        np_steps = max(1, min(e2e_steps, 5))
        for _ in range(2):
            nf.refine_type5(plan, ns, passes=PASSES)
            nf.refine_type4(plan, nA, passes=PASSES)
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(np_steps):
            y5 = nf.refine_type5(plan, ns, passes=PASSES)
            y4 = nf.refine_type4(plan, nA, passes=PASSES)
        np_s = max_over_ranks(time.perf_counter() - t0, world, dev, gloo)
        assert isinstance(y5, np.ndarray) and isinstance(y4, np.ndarray)
        e2e_np = {"value": pts_per_step * np_steps / np_s, "unit": "points/s", "h2d_bytes_per_step": bytes_io,
                  "d2h_bytes_per_step": bytes_io, "steps": np_steps,
                  "api": "refine_type5/refine_type4 on numpy arrays (the reference's convention; pageable memory)"}
        del ns, nA, y5, y4

    # ---- roofline of the dominant kernel (live per-launch events of the profiled pass)
    peaks_path = os.path.join(REPO, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        peak, peak_src = float(json.load(open(peaks_path))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    tfile = os.path.join(REPO, "profiles", f"traffic_{args.config}.json")
    tj = json.load(open(tfile)) if os.path.exists(tfile) and world == 1 and args.scaling == "strong" else {}

    def traffic_of(name):
        return tj.get(name, next((v for kk, v in tj.items() if kk.startswith(name + "_")), None))

    top = max(kprof.items(), key=lambda kv: kv[1][1]) if kprof else ("", (0, 0.0))
    tname, (tcount, tms) = top
    step_kernel_ms = sum(v[1] for v in kprof.values())
    roof = None
    if tname in ALGO_BYTES_PER_POINT_STEP and tcount:
        # algorithmic bytes per launch = (bytes/pt/step x points/step) / launches per step
        algo = ALGO_BYTES_PER_POINT_STEP[tname] * B * P * args.steps / tcount
        avg_ms = tms / tcount
        achieved = algo / (avg_ms / 1e3) / 1e9
        roof = {"kernel": tname, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic_of(tname), "algorithmic_bytes_per_launch": algo,
                "avg_launch_ms": avg_ms, "launches": tcount, "share_of_kernel_time": tms / step_kernel_ms,
                "peak_source": peak_src}
    per_kernel_roofline = {}
    for name, (cnt, kms) in kprof.items():
        if name in ALGO_BYTES_PER_POINT_STEP and kms > 0:
            gbs = ALGO_BYTES_PER_POINT_STEP[name] * B * P * args.steps / (kms / 1e3) / 1e9
            per_kernel_roofline[name] = {"achieved_GBps": gbs, "frac": gbs / peak}
            tb = traffic_of(name)
            if tb and cnt:
                dram = tb / (kms / cnt / 1e3) / 1e9
                per_kernel_roofline[name].update({"dram_GBps": dram, "dram_frac": dram / peak})
    total_algo = sum(ALGO_BYTES_PER_POINT_STEP[kk] for kk in kprof if kk in ALGO_BYTES_PER_POINT_STEP) * B * P
    step_s = ms / args.steps / 1e3
    line = {
        "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(cfg, world, args, signals_here=B, job=job,
                               extra={"damping_a": params.damping_a, "streams": args.streams}),
        "roofline": roof,
        "e2e": e2e,
        "e2e_numpy": e2e_np,
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "gather": gather,
        "plan_ms": plan_ms,
        "plan_warm_ms": plan_warm_ms,
        "plan_rebuild_ms_all": rebuild_ms,
        # single transforms (the plan is not amortised for C1, C3, C5):
        # the same metric with one warm plan build charged to every step
        "with_plan": ({"value": pts_per_step / ((ms / args.steps + plan_warm_ms) / 1e3), "unit": "points/s",
                       "ms_per_step": ms / args.steps + plan_warm_ms} if job == 1 else None),
        "parity": {"forward_residual_type5": resid5, "forward_residual_type4": resid4},
        "kernels_ms_per_step": {kk: v[1] / args.steps for kk, v in sorted(kernels_raw.items(), key=lambda kv: -kv[1][1])},
        "profiled_pass_ms_per_step": profiled_ms / args.steps,
        "kernel_roofline": per_kernel_roofline,
        "kernel_timing": kernel_timing,
        "step_roofline": {"algorithmic_bytes_per_step_per_gpu": total_algo,
                          "achieved_GBps": total_algo / step_s / 1e9,
                          "frac": total_algo / step_s / 1e9 / peak},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # bounded sample: one warm-up step and one timed step of one signal per host core
        ref, pts, secs, facts = cpu_reference_figures(cfg, 1, 1)
        line["cpu_baseline"] = {"value": pts / secs, "unit": "points/s", "cores": ref.cores, "kind": ref.kind,
                                "sample": ref.describe(job), "host": facts}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
