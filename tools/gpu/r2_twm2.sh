#!/bin/bash
# twisted row-modified sweep: parity (auto / forced), c5 timing default (auto), forced, forced + L2 hints
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "twisted or sweeps or step" > gpurun_out/pytest_twm2.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_twm2.log
for v in "auto|" "forced|ADI_SW_TWM=1" "forced_hint|ADI_SW_TWM=1 ADI_LIB=build/variants/twm_hint/libadimaxwell.so" "off|ADI_SW_TWM=0"; do
  name=${v%%|*}; envs=${v#*|}
  echo "== $name"
  env $envs timeout 300 python tools/profile_step.py --config c5 --steps 3 --timing 2>&1 | grep -E "sweep_mod|steps"
  env $envs timeout 300 python tools/profile_step.py --config c4 --steps 10 --timing 2>&1 | grep -E "sweep_mod|steps"
done
ADI_SW_TWM=1 ADI_LIB=build/variants/twm_hint/libadimaxwell.so timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:sweep_twm -c 1 python tools/profile_step.py --config c5 --steps 1 2>&1 | grep -E "dram__|gpu__time|lts__"
