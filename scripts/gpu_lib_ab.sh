# A/B of library builds on the C4 bench (kernel table from the profiled pass)
cd $GRAFT_REPO_ROOT
for i in 1 2; do
for L in ${LIBS:-libnfft45_base.so libnfft45.so}; do
NFFT45_LIB=$PWD/paper_1604_06236_b200/lib/$L python bench.py --no-cpu-baseline --no-e2e --steps 20 ${BENCH_ARGS} > gpurun_out/ab.json 2>/dev/null
LIBNAME=$L python -c "
import json, os; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']
print(os.environ['LIBNAME'], round(d['ms_per_step'],3), {n: round(v,3) for n,v in list(k.items())[:9]})"
done; done
