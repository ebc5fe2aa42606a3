#!/bin/bash
# ncu full set of the row-modified sweep, twisted vs one lane per fiber (c5)
mkdir -p gpurun_out
for k in 1 0; do
ADI_SW_TWM=$k timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sweep_twm|sweep_kernel" -c 2 \
  -o gpurun_out/twm$k -f python tools/profile_step.py --config c5 --steps 1 > gpurun_out/ncu_twm$k.log 2>&1; echo ncu$k=$?
ncu -i gpurun_out/twm$k.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,dram__throughput.avg.pct_of_peak_sustained_elapsed > gpurun_out/twm${k}_raw.csv
done
cat gpurun_out/twm1_raw.csv gpurun_out/twm0_raw.csv | cut -c1-400
