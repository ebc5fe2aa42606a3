# round 2 (re-entry): full ncu set + source page of the TMA sweeps (DER bootstrap, 2 MASS, fused DER) at c5
mkdir -p gpurun_out
python tools/profile_step.py --config c5 --steps 1 --timing > gpurun_out/plain_r2d.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:sweep_tma -c 3 \
    -o /tmp/prof_st -f python tools/profile_step.py --config c5 --steps 1 > gpurun_out/ncu_full_r2d_st.log 2>&1
echo rc=$?
ncu -i /tmp/prof_st.ncu-rep --page raw --csv > gpurun_out/raw_r2d_st.csv
ncu -i /tmp/prof_st.ncu-rep --page source --csv > gpurun_out/src_r2d_st.csv
cat gpurun_out/plain_r2d.log
