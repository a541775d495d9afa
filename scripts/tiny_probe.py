"""Small-P solves: one-CTA fused kernel (tiny.cu) vs the general path (NFFT45_NO_TINY=1),
device-resident, refined type-5 + type-4 per step, CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1604_06236_b200 as nf
for P, B in ((64, 1), (64, 1024), (128, 256), (256, 1), (256, 64), (256, 1024)):
    t = bench.make_nodes(P, 0.3, 7)
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2), device=0)
    x = torch.randn(B, P, dtype=torch.complex128, device="cuda")
    o5, o4 = torch.empty_like(x), torch.empty_like(x)
    for _ in range(3):
        nf.refine_type5(plan, x, passes=1, out=o5); nf.refine_type4(plan, x, passes=1, out=o4)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        nf.refine_type5(plan, x, passes=1, out=o5); nf.refine_type4(plan, x, passes=1, out=o4)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    print(f"{os.environ.get('NFFT45_NO_TINY') and 'general' or 'tiny   '} P={P:4d} B={B:5d}: {ms:7.4f} ms/step  {2*B*P/ms*1e3:.3e} pts/s", flush=True)
