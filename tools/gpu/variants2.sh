mkdir -p gpurun_out
for lib in default build/variants/*/libadimaxwell.so; do
  if [ "$lib" = default ]; then L=""; else L="$lib"; fi
  echo "== $lib c5"
  ADI_LIB=$L timeout 300 python tools/profile_step.py --config c5 --steps 2 --timing 2>&1 | grep -E "sweep|steps"
done
for b in 1; do
  echo "== default c5 ADI_SW_BPS_MASS=$b"
  ADI_SW_BPS_MASS=$b timeout 300 python tools/profile_step.py --config c5 --steps 2 --timing 2>&1 | grep -E "sweep_mass"
done
