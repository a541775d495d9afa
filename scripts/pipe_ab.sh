mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
for v in "NFFT45_PIPE_MIN_BYTES=0" "NFFT45_PIPE_MIN_BYTES=100000000000"; do
 for c in c1 c2 c3 c4; do
  env $v python bench.py --config $c --no-cpu-baseline > gpurun_out/pab_$c.log 2>&1
  python - $c "$v" <<'PY'
import json, sys
c = sys.argv[1]
d = json.loads(open(f"gpurun_out/pab_{c}.log").read().strip().splitlines()[-1])
print(sys.argv[2], c, f"{d['ms_per_step']:.4f} ms/step", f"value {d['value']:.3g}", f"e2e {d['e2e']['value']:.3g}", d["e2e"].get("warmup_steps"))
PY
 done
done
