# ncu evidence for the c5 step: launch list (cold, serialised) + full sets of substep 1.
mkdir -p gpurun_out
CFG=${CFG:-c5}
python tools/profile_step.py --config $CFG --steps 1 --timing > gpurun_out/plain_$CFG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv \
    python tools/profile_step.py --config $CFG --steps 1 > gpurun_out/ncu_launch_$CFG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sweep|rhs" -c ${NK:-24} \
    -o gpurun_out/prof_$CFG -f python tools/profile_step.py --config $CFG --steps 1 > gpurun_out/ncu_full_$CFG.log 2>&1
echo rc=$?
cat gpurun_out/plain_$CFG.log
