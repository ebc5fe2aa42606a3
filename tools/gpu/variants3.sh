#!/bin/bash
# time the sweep kernels of every tuning build under build/variants at c5 (plus the default)
mkdir -p gpurun_out
for lib in default build/variants/*/libadimaxwell.so; do
  if [ "$lib" = default ]; then L=""; else L="$lib"; fi
  echo "== $lib c5 $EXTRA_ENV"
  env ADI_LIB=$L $EXTRA_ENV timeout 300 python tools/profile_step.py --config c5 --steps 2 --timing 2>&1 | grep -E "sweep|steps"
done
