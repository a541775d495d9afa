# A/B of env-switch variants on the C4 bench (kernel table from the profiled pass).
# VARIANTS="NFFT45_HYB=0 NFFT45_FUSE=0" scripts/env_ab.sh   ("-" = default build)
cd $GRAFT_REPO_ROOT
for i in 1 2; do
for V in - ${VARIANTS}; do
if [ "$V" = "-" ]; then E=""; else E="$V"; fi
env $(echo $E | tr ',' ' ') python bench.py --no-cpu-baseline --no-e2e --steps 20 ${BENCH_ARGS} > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -5 gpurun_out/ab.err
VNAME="$V" python -c "
import json, os; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']
print(os.environ['VNAME'], round(d['ms_per_step'],3), {n: round(v,3) for n,v in list(k.items())[:9]})"
done; done
