"""One warm plan build (a fresh node-set handle, pooled memory) between cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists: usage  python scripts/plan_profile.py <log2 P> [eta].
Without ncu it prints the wall-clock time of warm builds (NFFT45_PLAN_TIMING=1 adds the host breakdown)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1604_06236_b200 as nf

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 20
eta = int(sys.argv[2]) if len(sys.argv) > 2 else bench.ETA
P = 1 << lg
t = bench.make_nodes(P, 0.3, 16043)
params = nf.MethodParams.from_mu(bench.MU, P, eta)
keep = nf.build_plan(nf.validate_grid(t), params, device=0)  # one-time costs (module load, twiddles)
times = []
for rep in range(5):
    g2 = nf.validate_grid(t)
    g2.device_handle(0)
    torch.cuda.synchronize()
    if rep == 4:
        torch.cuda.profiler.start()
    t0 = time.perf_counter()
    plan = nf.build_plan(g2, params, device=0)
    torch.cuda.synchronize()
    times.append(1e3 * (time.perf_counter() - t0))
    if rep == 4:
        torch.cuda.profiler.stop()
    del plan, g2
print(f"P=2^{lg} eta={eta}: warm plan builds {['%.3f' % x for x in times]} ms")
