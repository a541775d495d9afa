# A/B of programmatic dependent launch (NFFT45_NO_PDL=1 turns it off): bench lines per
# config, bitwise equality of refined outputs, then the GPU test suite with PDL on
mkdir -p gpurun_out
for c in c2 c3 c1 c4; do
  for e in "NFFT45_NO_PDL=1" "NFFT45_PDL_ON=1"; do
    env $e timeout 300 python bench.py --config $c 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '$e', round(d['ms_per_step'],4), '%.4g' % d['value'], 'e2e %.4g' % d['e2e']['value'])"
  done
done > gpurun_out/pdl_ab.log 2>&1
ENVSW=NFFT45_NO_PDL=1 bash scripts/ab_env.sh
[ -n "$NOTEST" ] || timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
