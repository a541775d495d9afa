"""One bench step (refined type-5 + refined type-4) between cudaProfilerStart/Stop, for
`ncu --profile-from-start off` captures: usage  python scripts/profile_step.py <c1|c2|c3|c4>."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1604_06236_b200 as nf

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
P, B = cfg["P"], cfg["B"]
t = bench.make_nodes(P, cfg["J"], cfg["seed"])
plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(bench.MU, P, bench.ETA), device=0)
g = torch.Generator(device="cuda:0")
g.manual_seed(cfg["seed"])
mk = lambda: torch.complex(torch.randn(B, P, generator=g, device="cuda:0", dtype=torch.float64),
                           torch.randn(B, P, generator=g, device="cuda:0", dtype=torch.float64)) / math.sqrt(2)
s, A = mk(), mk()
o5, o4 = torch.empty_like(s), torch.empty_like(A)
for _ in range(3):
    nf.refine_type5(plan, s, passes=bench.PASSES, out=o5)
    nf.refine_type4(plan, A, passes=bench.PASSES, out=o4)
torch.cuda.synchronize()
torch.cuda.profiler.start()
nf.refine_type5(plan, s, passes=bench.PASSES, out=o5)
nf.refine_type4(plan, A, passes=bench.PASSES, out=o4)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled one step of", cfg["label"])
