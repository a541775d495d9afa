set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/gputest.log
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"
tail -c 2500 gpurun_out/bench_c4.json
python tests/tools/c5_sweep.py > gpurun_out/c5.log 2>&1; echo "c5 rc=$?"
