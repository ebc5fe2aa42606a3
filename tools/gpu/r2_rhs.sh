#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or rhs or c1_full or c4_full" > gpurun_out/pytest_rhs.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_rhs.log
timeout 300 python tools/profile_step.py --config c5 --steps 2 --timing 2>&1 | tail -7
ADI_RHS3=0 timeout 300 python tools/profile_step.py --config c5 --steps 2 --timing 2>&1 | tail -7
timeout 300 python -m pytest tests/test_dist_gpu.py -x -q 2>&1 | tail -2
