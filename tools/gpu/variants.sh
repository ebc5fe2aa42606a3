# c5 / c4 step timing for each tuning build under build/variants (and the default build)
mkdir -p gpurun_out
for lib in default build/variants/*/libadimaxwell.so; do
  for cfg in c5 c4; do
    echo "== $lib $cfg"
    if [ "$lib" = default ]; then L=""; else L="$lib"; fi
    ADI_LIB=$L timeout 300 python tools/profile_step.py --config $cfg --steps 2 --timing 2>&1 | grep -E "sweep|rhs|steps"
  done
done
