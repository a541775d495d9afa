mkdir -p gpurun_out
for v in "X=1" "NFFT45_PIPE_ALT=1" "NFFT45_NO_GRAPH=1" "NFFT45_PIPE_ALT=1 NFFT45_NO_GRAPH=1"; do
 for c in c2 c3; do
  env $v python bench.py --config $c --no-cpu-baseline > gpurun_out/alt_$c.log 2>&1
  python - $c "$v" <<'PY'
import json, sys
c = sys.argv[1]
d = json.loads(open(f"gpurun_out/alt_{c}.log").read().strip().splitlines()[-1])
print(sys.argv[2], c, f"{d['ms_per_step']:.4f} ms/step", f"e2e {d['e2e']['value']:.3g}", d["e2e"].get("warmup_steps"))
PY
 done
done
