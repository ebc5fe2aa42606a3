# round 2: bench (ours + reference arm) and the ncu launch list of the same command
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_r2.txt
python bench.py > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; echo bench=$?
python bench.py --impl reference > gpurun_out/bench_ref_r2.json 2> gpurun_out/bench_ref_r2.err; echo ref=$?
python bench.py --config c4 --no-cpu-baseline > gpurun_out/bench_r2_c4.json 2> gpurun_out/bench_r2_c4.err; echo c4=$?
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_r2.log 2>&1; echo ncu=$?
cat gpurun_out/bench_r2.json
