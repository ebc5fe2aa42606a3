# full ncu set (with source) of NK launches matching REGEX in one step of CFG
mkdir -p gpurun_out
CFG=${CFG:-c5}; TAG=${TAG:-x}; REGEX=${REGEX:-rhs}; NK=${NK:-2}
python tools/profile_step.py --config $CFG --steps 1 --timing > gpurun_out/plain_${CFG}_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$REGEX" -c $NK \
    -o /tmp/prof_${CFG}_$TAG -f python tools/profile_step.py --config $CFG --steps 1 > gpurun_out/ncu_full_${CFG}_$TAG.log 2>&1
echo rc=$?
ncu -i /tmp/prof_${CFG}_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_${CFG}_$TAG.csv
ncu -i /tmp/prof_${CFG}_$TAG.ncu-rep --page source --csv > gpurun_out/src_${CFG}_$TAG.csv
sz=$(stat -c %s /tmp/prof_${CFG}_$TAG.ncu-rep); echo size=$sz
if [ "$sz" -lt 40000000 ]; then cp /tmp/prof_${CFG}_$TAG.ncu-rep gpurun_out/; fi
cat gpurun_out/plain_${CFG}_$TAG.log
