#!/bin/bash
# row-modified sweep register caps (ADI_SW_MINB_MOD = 3, 4 resident blocks), twisted and one lane per fiber
mkdir -p gpurun_out
for lib in "" build/variants/mod_minb3/libadimaxwell.so build/variants/mod_minb4/libadimaxwell.so; do
  for k in 1 0; do
    echo "== lib=${lib:-default} ADI_SW_TWM=$k"
    ADI_LIB=$lib ADI_SW_TWM=$k timeout 300 python tools/profile_step.py --config c5 --steps 3 --timing 2>&1 | grep -E "sweep_mod"
  done
done
