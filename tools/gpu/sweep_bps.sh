# c5/c4 step timing vs the sweep kernels' blocks-per-SM cap
mkdir -p gpurun_out
for cfg in c5 c4; do
for b in 1 2 3; do
  echo "== $cfg ADI_SW_BPS_MASS=$b ADI_SW_BPS_MOD=$b"
  ADI_SW_BPS_MASS=$b ADI_SW_BPS_MOD=$b timeout 300 python tools/profile_step.py --config $cfg --steps 2 --timing 2>&1 | grep sweep
done
done
