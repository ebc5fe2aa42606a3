#!/bin/bash
# row-modified sweep variants at c5: pivot recompute (default, occupancy grid and 1 block/SM) vs cached pivots
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "mod or sweep or parity" > gpurun_out/pytest_modvar.log 2>&1; echo pytest=$?
for v in "default|" "bps1|ADI_SW_BPS_MOD=1" "cached|ADI_LIB=build/variants/cached/libadimaxwell.so" "cached_bps1|ADI_LIB=build/variants/cached/libadimaxwell.so ADI_SW_BPS_MOD=1"; do
  name=${v%%|*}; envs=${v#*|}
  echo "== $name"
  env $envs timeout 300 python tools/profile_step.py --config c5 --steps 2 --timing 2>&1 | grep -E "sweep|steps"
done
