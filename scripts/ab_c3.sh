# A/B of the previous and the current library on single transforms (C3 / C5 sizes) and
# the bitwise-equality of their outputs; then the GPU test suite on the current one.
set -x
mkdir -p gpurun_out
LIBS="lib/libnfft45_old.so lib/libnfft45.so" CMD="python scripts/single_probe.py" bash scripts/lib_ab.sh > gpurun_out/ab_single.log 2>&1
for l in lib/libnfft45_old.so lib/libnfft45.so; do
  NFFT45_LIB=$PWD/paper_1604_06236_b200/$l python - >> gpurun_out/ab_bits.log 2>&1 <<'PY'
import os, sys, torch, hashlib
sys.path.insert(0, os.getcwd())
import bench, paper_1604_06236_b200 as nf
for P, B in [(1 << 20, 1), (1 << 18, 1), (4096, 4), (4096, 64)]:
    t = bench.make_nodes(P, 0.3, 7)
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2), device=0)
    g = torch.Generator().manual_seed(3)
    x = torch.randn(B, P, dtype=torch.complex128, generator=g).cuda()
    a = nf.refine_type5(plan, x, passes=1); b = nf.refine_type4(plan, x, passes=1)
    h = hashlib.sha1(torch.cat([a.flatten(), b.flatten()]).cpu().numpy().tobytes()).hexdigest()
    print(os.environ["NFFT45_LIB"].split("/")[-1], P, B, h, flush=True)
PY
done
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
