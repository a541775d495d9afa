for l in lib/libnfft45_old.so lib/libnfft45_new.so; do
 for v in "X=1" "NFFT45_NO_GRAPH=1"; do
  env $v NFFT45_LIB=$PWD/paper_1604_06236_b200/$l python bench.py --config c1 --no-cpu-baseline > gpurun_out/c1ab.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/c1ab.log').read().strip().splitlines()[-1]);print('$l $v', d['ms_per_step'], d['plan_warm_ms'])"
 done
done
