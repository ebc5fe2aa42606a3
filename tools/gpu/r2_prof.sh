# round 2: full ncu sets of the top kernels at c5 (one launch each), raw + source pages
mkdir -p gpurun_out
python tools/profile_step.py --config c5 --steps 1 --timing > gpurun_out/plain_r2.log 2>&1 || exit 1
for k in rhs3 sweep_tma; do
  ncu --set full --clock-control none --import-source on -k regex:"$k" -c ${NK:-1} \
      -o /tmp/prof_$k -f python tools/profile_step.py --config c5 --steps 1 > gpurun_out/ncu_full_$k.log 2>&1
  echo $k rc=$?
  ncu -i /tmp/prof_$k.ncu-rep --page raw --csv > gpurun_out/raw_r2_$k.csv
  ncu -i /tmp/prof_$k.ncu-rep --page source --csv > gpurun_out/src_r2_$k.csv
  ncu -i /tmp/prof_$k.ncu-rep --page details --csv > gpurun_out/det_r2_$k.csv
done
cat gpurun_out/plain_r2.log
