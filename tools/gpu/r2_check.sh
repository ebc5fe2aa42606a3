#!/bin/bash
# round-2 GPU check: selected parity tests, then the c5 bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -k "${PYTEST_K:-golden or singular or c1_full}" > gpurun_out/pytest_sel.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_sel.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench=$?
cat gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5.err
