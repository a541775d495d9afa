#!/usr/bin/env python
"""Single-signal refined type-5 + type-4 step time across P (chain vs generic sizes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1604_06236_b200 as nf
for P in [1 << 14, 1 << 15, 1 << 16, 1 << 17, 1 << 18, 1 << 19, 1 << 20, 3 << 16, 100000]:
    t = bench.make_nodes(P, 0.3, 7)
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2), device=0)
    x = torch.randn(P, dtype=torch.complex128, device="cuda")
    o5, o4 = torch.empty_like(x), torch.empty_like(x)
    for _ in range(3):
        nf.refine_type5(plan, x, passes=1, out=o5); nf.refine_type4(plan, x, passes=1, out=o4)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        nf.refine_type5(plan, x, passes=1, out=o5); nf.refine_type4(plan, x, passes=1, out=o4)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"P={P:8d}: {ms:7.3f} ms/step  {2*P/ms*1e3:.3e} pts/s", flush=True)
