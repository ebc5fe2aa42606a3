#!/bin/bash
# twisted row-modified sweep: parity, then c5 per-class timing with and without it
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "twisted or sweeps or rhs_and_solve or step" > gpurun_out/pytest_twm.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_twm.log
for k in 1 0; do
  echo "== ADI_SW_TWM=$k"
  ADI_SW_TWM=$k timeout 300 python tools/profile_step.py --config c5 --steps 3 --timing 2>&1 | grep -E "sweep|rhs|steps"
done
ADI_SW_TWM=1 timeout 300 python tools/profile_step.py --config c4 --steps 10 --timing 2>&1 | grep -E "sweep_mod|steps"
ADI_SW_TWM=0 timeout 300 python tools/profile_step.py --config c4 --steps 10 --timing 2>&1 | grep -E "sweep_mod|steps"
