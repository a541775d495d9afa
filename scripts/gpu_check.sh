# full GPU test suite + smoke + bench lines for every config (run under gpurun)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in ${CONFIGS:-c4 c3 c2 c1}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
  python - $c <<'PY'
import json, sys
c = sys.argv[1]
d = json.loads(open(f"gpurun_out/bench_{c}.log").read().strip().splitlines()[-1])
rf = d.get("roofline") or {}
print(c, f"{d['ms_per_step']:.4f} ms/step", f"value {d['value']:.3g}", f"e2e {d['e2e']['value']:.3g}",
      rf.get("kernel"), rf.get("frac"), d["e2e"].get("warmup_steps"))
PY
done
