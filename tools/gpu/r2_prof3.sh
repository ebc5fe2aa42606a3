# round 2 final: full ncu sets of the step's kernels at c5: rhs3 (1), sweep_tma (bootstrap DER, 2 mass, fused DER), sweep_kernel (MOD, 1)
mkdir -p gpurun_out
python tools/profile_step.py --config c5 --steps 1 --timing > gpurun_out/plain_r2c.log 2>&1 || exit 1
for spec in "rhs3:1" "sweep_tma:4" "sweep_kernel:1"; do
  k=${spec%%:*}; c=${spec##*:}
  ncu --set full --clock-control none --import-source on -k regex:"$k" -c $c \
      -o /tmp/prof_$k -f python tools/profile_step.py --config c5 --steps 1 > gpurun_out/ncu_full_r2c_$k.log 2>&1
  echo $k rc=$?
  ncu -i /tmp/prof_$k.ncu-rep --page raw --csv > gpurun_out/raw_r2c_$k.csv
  ncu -i /tmp/prof_$k.ncu-rep --page source --csv > gpurun_out/src_r2c_$k.csv
done
cat gpurun_out/plain_r2c.log
