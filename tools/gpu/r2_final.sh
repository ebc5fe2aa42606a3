# round 2 final: GPU suite (driver command), smoke, bench (ours, reference arm, c4), ncu launch list + full sets
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/final_pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/final_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/final_smoke.log
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench=$?
python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo ref=$?
python bench.py --config c4 --no-cpu-baseline > gpurun_out/final_bench_c4.json 2> gpurun_out/final_bench_c4.err; echo c4=$?
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final_bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final_ncu_launch.log 2>&1; echo ncu_launch=$?
bash tools/gpu/r2_prof3.sh > gpurun_out/final_prof.log 2>&1; echo prof=$?
cat gpurun_out/final_bench.json
