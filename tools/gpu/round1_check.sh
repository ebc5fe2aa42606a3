mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
ls -la --time-style=full-iso paper_2103_06998_b200/lib paper_2103_06998_b200/csrc
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench=$?
timeout 600 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench4=$?
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench_c5.json gpurun_out/bench_c4.json; tail -5 gpurun_out/bench_c5.err
