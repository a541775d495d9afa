cd $GRAFT_REPO_ROOT
nproc; lscpu | grep -E "Model name|Socket|Thread|Core|NUMA" 
for T in 8 12 16; do
NFFT45_COPY_THREADS=$T python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_np$T.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/bench_np$T.json').read().strip().splitlines()[-1]); print('$T threads', d['e2e_numpy']['value'], d['e2e']['value'])"
done
