#!/usr/bin/env python
"""e2e probe: C4 step through the public API with pinned host buffers (as bench.py's e2e)."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1604_06236_b200 as nf
P, B = 1 << 16, 1024
NB = os.environ.get('NB', '0') == '1'
t = bench.make_nodes(P, 0.3, 16044)
grid = nf.validate_grid(t)
plan = nf.build_plan(grid, nf.MethodParams.from_mu(1e-15, P, 2), device=0)
hs = (torch.randn(B, P, dtype=torch.complex128) ).pin_memory()
hA = (torch.randn(B, P, dtype=torch.complex128) ).pin_memory()
o5, o4 = torch.empty_like(hs).pin_memory(), torch.empty_like(hA).pin_memory()
nf.refine_type5(plan, hs, passes=1, out=o5); torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    for _ in range(3):
        nf.refine_type5(plan, hs, passes=1, out=o5, non_blocking=NB)
        nf.refine_type4(plan, hA, passes=1, out=o4, non_blocking=NB)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"nb {NB} chunk {os.environ.get('NFFT45_STREAM_CHUNK', '64')}: {dt*1e3:.1f} ms/step  e2e {2*B*P/dt:.3e} pts/s", flush=True)
