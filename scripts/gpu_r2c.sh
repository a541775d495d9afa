cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_reference_semantics.py tests/test_gpu_parity.py tests/test_gpu_cli_bench.py -m gpu -q -p no:cacheprovider -k "numpy_operands or harness or multi_pass" > gpurun_out/gputest_d.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/gputest_d.log
python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_np.json 2> gpurun_out/bench_np.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_np.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step']); print(d['e2e']); print(d['e2e_numpy'])"
NFFT45_COPY_THREADS=4 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_np4.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/bench_np4.json').read().strip().splitlines()[-1]); print('4 threads', d['e2e_numpy'])"
