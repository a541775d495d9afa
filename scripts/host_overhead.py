"""Host-side cost per Python call of a tiny solve (P = 64, device tensors, out= given)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1604_06236_b200 as nf
P = 64
plan = nf.build_plan(nf.validate_grid(bench.make_nodes(P, 0.3, 1)), nf.MethodParams.from_mu(1e-15, P, 2), device=0)
x = torch.randn(P, dtype=torch.complex128, device="cuda")
o = torch.empty_like(x)
for _ in range(100):
    nf.refine_type5(plan, x, passes=1, out=o)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(2000):
    nf.refine_type5(plan, x, passes=1, out=o)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host time per call {1e6*(t1-t0)/2000:.1f} us; with device drain {1e6*(time.perf_counter()-t0)/2000:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(2000):
    nf.refine_type5(plan, x, passes=1, out=o)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
