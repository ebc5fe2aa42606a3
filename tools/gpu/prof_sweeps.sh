# full ncu sets of the six sweep launches of substep 1 (CFG=c5|c4)
mkdir -p gpurun_out
CFG=${CFG:-c5}; TAG=${TAG:-x}
python tools/profile_step.py --config $CFG --steps 1 --timing > gpurun_out/plain_${CFG}_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sweep" -c ${NK:-6} \
    -o /tmp/prof_${CFG}_$TAG -f python tools/profile_step.py --config $CFG --steps 1 > gpurun_out/ncu_full_${CFG}_$TAG.log 2>&1
echo rc=$?
ncu -i /tmp/prof_${CFG}_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_${CFG}_$TAG.csv
sz=$(stat -c %s /tmp/prof_${CFG}_$TAG.ncu-rep); echo size=$sz
if [ "$sz" -lt 40000000 ]; then cp /tmp/prof_${CFG}_$TAG.ncu-rep gpurun_out/; fi
cat gpurun_out/plain_${CFG}_$TAG.log
