# round 2: full ncu sets (one launch each) of the fused RHS_E and the row-modified sweep at c5
mkdir -p gpurun_out
python tools/profile_step.py --config c5 --steps 1 --timing > gpurun_out/plain_r2b.log 2>&1 || exit 1
for k in ${KERNELS:-rhs3 sweep_kernel}; do
  ncu --set full --clock-control none --import-source on -k regex:"$k" -c 1 \
      -o /tmp/prof_$k -f python tools/profile_step.py --config c5 --steps 1 > gpurun_out/ncu_full_$k.log 2>&1
  echo $k rc=$?
  ncu -i /tmp/prof_$k.ncu-rep --page raw --csv > gpurun_out/raw_${TAG:-r2b}_$k.csv
  ncu -i /tmp/prof_$k.ncu-rep --page source --csv > gpurun_out/src_${TAG:-r2b}_$k.csv
done
cat gpurun_out/plain_r2b.log
