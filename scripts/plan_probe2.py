import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_1604_06236_b200 as nf
for P, J in ((1 << 20, 0.4), (1 << 16, 0.3)):
    t = bench.make_nodes(P, J, 16043)
    params = nf.MethodParams.from_mu(1e-15, P, 2)
    keep = []
    for rep in range(4):
        g2 = nf.validate_grid(t); g2.device_handle(0); torch.cuda.synchronize()
        t3 = time.perf_counter(); plan = nf.build_plan(g2, params); torch.cuda.synchronize(); t4 = time.perf_counter()
        keep.append(plan)
        t5 = time.perf_counter(); keep.pop(0) if len(keep) > 1 else None; torch.cuda.synchronize(); t6 = time.perf_counter()
        print(f"P={P} build {1e3*(t4-t3):.3f} ms, destroy {1e3*(t6-t5):.3f} ms", flush=True)
