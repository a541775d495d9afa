cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "variants_bitwise or c4_shape or c2_batched or rectangular_batch or three_times" > gpurun_out/gputest_tma.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/gputest_tma.log
for i in 1 2; do
for V in "" "NFFT45_NO_TMA=1"; do
env $V python bench.py --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/ab.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']
print('$V', round(d['ms_per_step'],3), {n: round(v,3) for n,v in k.items()})"
done; done
