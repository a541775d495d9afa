mkdir -p gpurun_out
for i in 1 2; do python bench.py --no-cpu-baseline > gpurun_out/b$i.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/b$i.log').read().strip().splitlines()[-1]);print('$i',d['ms_per_step'],'%.3g'%d['value'],'e2e %.3g'%d['e2e']['value'])"; done
python bench.py --no-cpu-baseline --e2e-steps 10 > gpurun_out/b3.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/b3.log').read().strip().splitlines()[-1]);print('e2e10',d['ms_per_step'],'%.3g'%d['value'],'e2e %.3g'%d['e2e']['value'])"
