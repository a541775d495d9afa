python scripts/profile_step.py c4 > gpurun_out/plain_step.log 2>&1 || exit 1
for K in kbm_band kbm_pad k_spread_p k_gather_p; do K=$K bash scripts/gpu_src.sh > /dev/null 2>&1; done
for K in kbm_band kbm_pad k_spread_p k_gather_p; do echo "== $K"; python scripts/sass_hot.py gpurun_out/src_${K}_sass.csv 25; done
