"""Device-resident refined type-5 + type-4 step at P = 2^16 across batch sizes (C4 shape),
CUDA events; writes profiles/batch_sweep.md."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1604_06236_b200 as nf
P = 1 << 16
t = bench.make_nodes(P, 0.3, 16044)
plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2), device=0)
rows = []
for B in (1, 4, 16, 64, 128, 256, 512, 1024, 2048):
    x = torch.randn(B, P, dtype=torch.complex128, device="cuda")
    o5, o4 = torch.empty_like(x), torch.empty_like(x)
    for _ in range(3):
        nf.refine_type5(plan, x, passes=1, out=o5); nf.refine_type4(plan, x, passes=1, out=o4)
    torch.cuda.synchronize()
    reps = max(3, min(50, 4096 // B))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        nf.refine_type5(plan, x, passes=1, out=o5); nf.refine_type4(plan, x, passes=1, out=o4)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    rows.append((B, ms, 2 * B * P / ms * 1e3, ms * 1e3 / B))
    print(f"B={B:5d}: {ms:8.3f} ms/step  {rows[-1][2]:.3e} pts/s  {rows[-1][3]:.1f} us/signal", flush=True)
    del x, o5, o4
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/batch_sweep.md", "w") as f:
    f.write("# Batch sweep at P = 2^16 (C4 shape), B200, refined type-5 + type-4 per step, device-resident\n\n")
    f.write("`python scripts/batch_sweep.py`. Batches below 16 run the signal-major chains, 16 and up the batch-minor ones.\n\n")
    f.write("| signals | ms/step | points/s | us per signal |\n|---|---|---|---|\n")
    for B, ms, v, us in rows:
        f.write(f"| {B} | {ms:.3f} | {v:.3e} | {us:.1f} |\n")
