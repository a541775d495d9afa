# per-CUDA-source-line instruction counts and stalls of one launch of kernel $K (regex), config $CFG
mkdir -p gpurun_out
python scripts/profile_step.py ${CFG:-c4} > /dev/null 2>&1 || exit 1
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$K --launch-skip ${SKIP:-0} -c 1 \
    -o gpurun_out/srcc_${K} -f python scripts/profile_step.py ${CFG:-c4} > gpurun_out/srcc_${K}.log 2>&1
ncu -i gpurun_out/srcc_${K}.ncu-rep --page source --csv --print-source cuda > gpurun_out/srcc_${K}_cuda.csv 2>>gpurun_out/srcc_${K}.log
ncu -i gpurun_out/srcc_${K}.ncu-rep --page source --csv --print-source sass > gpurun_out/srcc_${K}_sass.csv 2>>gpurun_out/srcc_${K}.log
rm -f gpurun_out/srcc_${K}.ncu-rep
