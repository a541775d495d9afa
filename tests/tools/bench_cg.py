"""CG baseline throughput: GPU CGNR vs the fast inverse
(refine_type4) and the CPU oracle CGNR on the same type-4 systems."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_1604_06236_b200 as nf
from oracle import nfft_oracle as O

for P, J in ((4096, 0.3), (1 << 16, 0.3), (1 << 16, 0.45)):
    t, data = O.make_inputs(P, J, 1, 77)
    grid = nf.validate_grid(t)
    a_true = data[0]
    b = nf.nfft_type1(grid, a_true, P)
    bd = torch.from_numpy(b).cuda()
    nf.cg_solve(grid, bd, "type4", tol=1e-12)  # warm-up
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = nf.cg_solve(grid, bd, "type4", tol=1e-12)
    torch.cuda.synchronize(); tg = time.perf_counter() - t0
    plan = nf.build_plan(grid, nf.MethodParams.from_mu(1e-15, P, 2))
    nf.refine_type4(plan, bd, passes=1); torch.cuda.synchronize()
    t0 = time.perf_counter(); x4 = nf.refine_type4(plan, bd, passes=1); torch.cuda.synchronize()
    tf = time.perf_counter() - t0
    err_cg = nf.relative_error(a_true, res.solution.cpu().numpy())
    err_f = nf.relative_error(a_true, x4.cpu().numpy())
    line = (f"P={P} J={J}: GPU CG {res.iterations} it, {tg*1e3:.1f} ms ({tg/max(res.iterations,1)*1e6:.0f} us/it), "
            f"err {err_cg:.1e} | fast refine_type4 {tf*1e3:.2f} ms err {err_f:.1e}")
    if P <= 4096:
        t0 = time.perf_counter(); x, it, conv, _ = O.cg(t, b, "type4", 1e-12); to = time.perf_counter() - t0
        line += f" | CPU oracle CG {it} it {to*1e3:.0f} ms"
    print(line, flush=True)
