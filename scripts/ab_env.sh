# A/B of an environment switch ($ENVSW, e.g. NFFT45_STILE=128) on single transforms and the
# bitwise equality of refined outputs with and without it
mkdir -p gpurun_out
for e in "" "$ENVSW"; do
  echo "== env: $e" >> gpurun_out/ab_env.log
  env $e python scripts/single_probe.py >> gpurun_out/ab_env.log 2>&1
  env $e python - >> gpurun_out/ab_env_bits.log 2>&1 <<'PY'
import os, sys, torch, hashlib
sys.path.insert(0, os.getcwd())
import bench, paper_1604_06236_b200 as nf
for P, B in [(1 << 20, 1), (1 << 18, 1), (4096, 4), (1000, 1)]:
    t = bench.make_nodes(P, 0.3, 7)
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2), device=0)
    g = torch.Generator().manual_seed(3)
    x = torch.randn(B, P, dtype=torch.complex128, generator=g).cuda()
    a = nf.refine_type5(plan, x, passes=1); b = nf.refine_type4(plan, x, passes=1)
    h = hashlib.sha1(torch.cat([a.flatten(), b.flatten()]).cpu().numpy().tobytes()).hexdigest()
    print(repr(os.environ.get("NFFT45_STILE")), P, B, h, flush=True)
PY
done
