#!/bin/bash
# A/B of env switches on the C4 bench: scripts/ab.sh "" "NFFT45_E8=1" ...
for v in "$@"; do
  env $v python bench.py --no-cpu-baseline --e2e-steps 1 --steps 10 > gpurun_out/ab.log 2>&1
  python - "$v" <<'PY'
import json,sys
d=json.loads(open("gpurun_out/ab.log").read().strip().splitlines()[-1])
k=d["kernels_ms_per_step"]
print(f"[{sys.argv[1] or 'default'}] {d['ms_per_step']:.3f} ms/step resid {d['parity']['forward_residual_type5']:.1e}/{d['parity']['forward_residual_type4']:.1e} ::", " ".join(f"{a}={b:.3f}" for a,b in k.items() if b>0.05))
PY
done
