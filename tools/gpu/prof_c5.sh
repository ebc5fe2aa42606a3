# ncu evidence for one step: launch list (cold, serialised) + full sets of the first NK launches.
mkdir -p gpurun_out
CFG=${CFG:-c5}
TAG=${TAG:-r1}
python tools/profile_step.py --config $CFG --steps 1 --timing > gpurun_out/plain_$CFG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}_$TAG.csv \
    python tools/profile_step.py --config $CFG --steps 1 > gpurun_out/ncu_launch_$CFG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sweep|rhs" -c ${NK:-15} \
    -o /tmp/prof_${CFG}_$TAG -f python tools/profile_step.py --config $CFG --steps 1 > gpurun_out/ncu_full_$CFG.log 2>&1
echo rc=$?
ncu -i /tmp/prof_${CFG}_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_${CFG}_$TAG.csv
ncu -i /tmp/prof_${CFG}_$TAG.ncu-rep --page details --csv > gpurun_out/details_${CFG}_$TAG.csv
ls -la /tmp/prof_${CFG}_$TAG.ncu-rep
sz=$(stat -c %s /tmp/prof_${CFG}_$TAG.ncu-rep)
if [ "$sz" -lt 45000000 ]; then cp /tmp/prof_${CFG}_$TAG.ncu-rep gpurun_out/; fi
cat gpurun_out/plain_$CFG.log
