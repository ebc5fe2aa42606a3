#!/bin/bash
# row-modified sweep on the TMA-staged kernel (ADI_SW_TMA bit 1) vs the cp.async default, c5 timing per class
mkdir -p gpurun_out
for v in "default|" "tma_w4r4|ADI_SW_TMA=7" "tma_w2r8|ADI_SW_TMA=7 ADI_LIB=build/variants/stm_w2r8/libadimaxwell.so" "tma_w6r3|ADI_SW_TMA=7 ADI_LIB=build/variants/stm_w6r3/libadimaxwell.so"; do
  name=${v%%|*}; envs=${v#*|}
  echo "== $name"
  env $envs timeout 300 python tools/profile_step.py --config c5 --steps 3 --timing 2>&1 | grep -E "sweep|rhs|steps"
done
ADI_SW_TMA=7 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep or step" 2>&1 | tail -2
