#!/usr/bin/env python
"""Experiment: does walking the C4 batch in L2-sized chunks beat one
full-batch solve?  Times one bench step (refined type-5 + refined type-4 over
1024 x 2^16) issued as 1024/Bc chunk solves, for several chunk sizes Bc, and
the interleaved order (type-5 chunk i, type-4 chunk i)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("NFFT45_NO_GRAPH", "1")

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1604_06236_b200 as nf  # noqa: E402

P, B = 1 << 16, 1024
t = bench.make_nodes(P, 0.3, 16044)
grid = nf.validate_grid(t)
params = nf.MethodParams.from_mu(1e-15, P, 2)
plan = nf.build_plan(grid, params, device=0)
g = torch.Generator(device="cuda:0")
g.manual_seed(1)
s = torch.complex(torch.randn(B, P, generator=g, device="cuda:0", dtype=torch.float64),
                  torch.randn(B, P, generator=g, device="cuda:0", dtype=torch.float64)) / math.sqrt(2)
A = torch.complex(torch.randn(B, P, generator=g, device="cuda:0", dtype=torch.float64),
                  torch.randn(B, P, generator=g, device="cuda:0", dtype=torch.float64)) / math.sqrt(2)
o5, o4 = torch.empty_like(s), torch.empty_like(A)


def step(bc, inter):
    if inter:
        for lo in range(0, B, bc):
            nf.refine_type5(plan, s[lo:lo + bc], passes=1, out=o5[lo:lo + bc])
            nf.refine_type4(plan, A[lo:lo + bc], passes=1, out=o4[lo:lo + bc])
    else:
        for lo in range(0, B, bc):
            nf.refine_type5(plan, s[lo:lo + bc], passes=1, out=o5[lo:lo + bc])
        for lo in range(0, B, bc):
            nf.refine_type4(plan, A[lo:lo + bc], passes=1, out=o4[lo:lo + bc])


for bc in [int(x) for x in (sys.argv[1:] or ["1024", "256", "128", "64", "32", "16"])]:
    for inter in (False, True):
        for _ in range(2):
            step(bc, inter)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            step(bc, inter)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"chunk {bc:5d} {'interleaved' if inter else 'sequential '}: {ms:7.2f} ms/step  "
              f"{2 * B * P / ms / 1e6:.3e} pts/s", flush=True)
