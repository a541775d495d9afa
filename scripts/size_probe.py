#!/usr/bin/env python
"""Throughput of the refined type-5 + type-4 step for sizes off the fused-chain
grid (P = M^2 powers of two use the chains; others take the generic path)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1604_06236_b200 as nf
cases = [(1 << 16, 256), (1 << 17, 128), (1 << 15, 512), (3 << 14, 256), (1 << 18, 32), (1 << 19, 16), (100000, 64), (4096, 64), (2048, 128)]
for P, B in cases:
    t = bench.make_nodes(P, 0.3, 7)
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2), device=0)
    x = torch.randn(B, P, dtype=torch.complex128, device="cuda")
    o5, o4 = torch.empty_like(x), torch.empty_like(x)
    for _ in range(2):
        nf.refine_type5(plan, x, passes=1, out=o5); nf.refine_type4(plan, x, passes=1, out=o4)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        nf.refine_type5(plan, x, passes=1, out=o5); nf.refine_type4(plan, x, passes=1, out=o4)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"P={P:7d} B={B:4d}: {ms:8.3f} ms/step  {2*B*P/ms/1e6:.3e} pts/s", flush=True)
