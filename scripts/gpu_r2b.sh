set -x
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_cli_bench.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "harness or multi_pass or in_place or 65535 or graph_cache or c4_shape or c2_batched" > gpurun_out/gputest_b.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/gputest_b.log
python -m pytest tests/test_gpu_reference_semantics.py -m gpu -q -p no:cacheprovider -k "in_place or 65535 or graph_cache" > gpurun_out/gputest_c.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/gputest_c.log
