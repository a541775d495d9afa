# source-level ncu page for one launch of kernel $K (regex) in config $CFG
mkdir -p gpurun_out
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$K --launch-skip ${SKIP:-0} -c 1 \
    -o gpurun_out/src_${K}${SKIP} -f python scripts/profile_step.py ${CFG:-c4} > gpurun_out/src_${K}${SKIP}.log 2>&1
ncu -i gpurun_out/src_${K}${SKIP}.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${K}${SKIP}_sass.csv 2>>gpurun_out/src_${K}${SKIP}.log
ncu -i gpurun_out/src_${K}${SKIP}.ncu-rep --page source --csv > gpurun_out/src_${K}${SKIP}_cuda.csv 2>>gpurun_out/src_${K}${SKIP}.log
ncu -i gpurun_out/src_${K}${SKIP}.ncu-rep --page raw --csv > gpurun_out/src_${K}${SKIP}_raw.csv 2>>gpurun_out/src_${K}${SKIP}.log
rm -f gpurun_out/src_${K}${SKIP}.ncu-rep
ls -la gpurun_out/src_*
