# ncu evidence of one c5 step (the bench workload): launch list + full sets of the first 11 launches
mkdir -p gpurun_out
CFG=${CFG:-c5}; TAG=${TAG:-r1}
python tools/profile_step.py --config $CFG --steps 1 > gpurun_out/plain_${CFG}_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}_$TAG.csv \
    python tools/profile_step.py --config $CFG --steps 1 > gpurun_out/ncu_launch_${CFG}_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel|rhs_kernel" -c 11 \
    -o /tmp/prof_${CFG}_$TAG -f python tools/profile_step.py --config $CFG --steps 1 > gpurun_out/ncu_full_${CFG}_$TAG.log 2>&1
echo rc=$?
ncu -i /tmp/prof_${CFG}_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_${CFG}_$TAG.csv
ncu -i /tmp/prof_${CFG}_$TAG.ncu-rep --page details --csv > gpurun_out/details_${CFG}_$TAG.csv
ncu -i /tmp/prof_${CFG}_$TAG.ncu-rep --page source --csv > gpurun_out/src_${CFG}_$TAG.csv
sz=$(stat -c %s /tmp/prof_${CFG}_$TAG.ncu-rep); echo size=$sz
if [ "$sz" -lt 30000000 ]; then cp /tmp/prof_${CFG}_$TAG.ncu-rep gpurun_out/; fi
tail -3 gpurun_out/ncu_full_${CFG}_$TAG.log
