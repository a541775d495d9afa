for i in 1 2 3; do python bench.py --config c2 --no-cpu-baseline > gpurun_out/c2_$i.log 2>&1; done
python bench.py --config c2 --no-cpu-baseline --streams 1 > gpurun_out/c2_s1.log 2>&1
python bench.py --config c2 --no-cpu-baseline --steps 50 > gpurun_out/c2_50.log 2>&1
for f in gpurun_out/c2_*.log; do python -c "
import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f','%.3g'%d['e2e']['value'],d['e2e']['steps'],d['e2e'].get('warmup_steps'))"; done
