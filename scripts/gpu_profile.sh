# ncu evidence for one bench step of each config (run under gpurun; one GPU)
mkdir -p gpurun_out
for c in ${CONFIGS:-c3 c4}; do
  python scripts/profile_step.py $c > gpurun_out/prof_$c.log 2>&1 || exit 1
  [ -n "$FULL_ONLY" ] || ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_$c.csv python scripts/profile_step.py $c >> gpurun_out/prof_$c.log 2>&1
  ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:^k \
      -o gpurun_out/full_$c -f python scripts/profile_step.py $c >> gpurun_out/prof_$c.log 2>&1
  ncu -i gpurun_out/full_$c.ncu-rep --page raw --csv > gpurun_out/full_$c.csv 2>> gpurun_out/prof_$c.log
  ncu -i gpurun_out/full_$c.ncu-rep --page details > gpurun_out/full_${c}_details.txt 2>> gpurun_out/prof_$c.log
  [ -n "$KEEP_REP" ] || rm -f gpurun_out/full_$c.ncu-rep
done
ls -la gpurun_out
