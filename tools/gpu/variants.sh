#!/bin/bash
# time the kernels of every tuning build under build/variants at c5 (plus the default build)
mkdir -p gpurun_out
for lib in default build/variants/*/libadimaxwell.so; do
  if [ "$lib" = default ]; then L=""; else L="$lib"; fi
  echo "== $lib ${CFG:-c5} $EXTRA_ENV"
  env ADI_LIB=$L $EXTRA_ENV timeout 300 python tools/profile_step.py --config ${CFG:-c5} --steps 2 --timing 2>&1 | grep -E "sweep|rhs|steps|Error|error"
done
