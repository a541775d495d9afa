"""Forward NFFT (nfft_type1 / nfft_type2, the reference's forward.py:26-102 entry points) timed on the
bench shapes, device-resident operands, with the per-kernel table of a profiled pass.
usage: python scripts/forward_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1604_06236_b200 as nf
from paper_1604_06236_b200 import _lib

dev = 0
SHAPES = ((1 << 16, 1024, 0.3), (1 << 12, 64, 0.3), (1 << 20, 1, 0.4))
for P, B, J in SHAPES[: int(os.environ.get("FWD_SHAPES", "3"))]:
    grid = nf.validate_grid(bench.make_nodes(P, J, 16044))
    g = torch.Generator(device=f"cuda:{dev}")
    g.manual_seed(7)
    x = torch.complex(torch.randn(B, P, generator=g, device=f"cuda:{dev}", dtype=torch.float64),
                      torch.randn(B, P, generator=g, device=f"cuda:{dev}", dtype=torch.float64))
    if B == 1:
        x = x[0]
    for name, fn in (("type1", lambda: nf.nfft_type1(grid, x, P)), ("type2", lambda: nf.nfft_type2(x, grid))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        reps = 5 if B >= 1024 else 30
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        _lib.profile_enable(True)
        fn()
        torch.cuda.synchronize()
        _lib.profile_enable(False)
        prof = _lib.profile_read()
        tab = {k: round(v[1], 4) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])}
        print(f"P={P} batch={B} {name}: {ms:.4f} ms  {P * B / ms / 1e6:.2f}e9 points/s  {tab}", flush=True)
