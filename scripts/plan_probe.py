#!/usr/bin/env python
"""Where does plan build time go? Wall time of build_plan (device grid
already uploaded) vs the sum of its kernel times (C-ABI launch profiler)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1604_06236_b200 as nf
from paper_1604_06236_b200 import _lib
for P, J in ((1 << 20, 0.4), (1 << 16, 0.3), (1 << 18, 0.3)):
    t = bench.make_nodes(P, J, 16043)
    t0 = time.perf_counter(); grid = nf.validate_grid(t); t1 = time.perf_counter()
    grid.device_handle(0); torch.cuda.synchronize(); t2 = time.perf_counter()
    params = nf.MethodParams.from_mu(1e-15, P, 2)
    for rep in range(3):
        g2 = nf.validate_grid(t); g2.device_handle(0); torch.cuda.synchronize()
        _lib.profile_enable(True)
        t3 = time.perf_counter(); plan = nf.build_plan(g2, params); torch.cuda.synchronize(); t4 = time.perf_counter()
        _lib.profile_enable(False)
        prof = _lib.profile_read()
        ks = sum(v[1] for v in prof.values())
        print(f"P={P} validate {1e3*(t1-t0):.1f} ms, grid upload {1e3*(t2-t1):.1f} ms, build_plan {1e3*(t4-t3):.1f} ms "
              f"(kernels {ks:.2f} ms): " + ", ".join(f"{k}={v[1]:.2f}" for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])[:8]), flush=True)
