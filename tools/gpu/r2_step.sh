# round 2: distributed (loopback) tests incl. the partitioned z-solve, RHS parity, c5 timing
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_dist_gpu.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo dist=$?
tail -5 gpurun_out/pytest_dist.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "rhs or fused or c1_full or c3_full or c4_full" > gpurun_out/pytest_rhs.log 2>&1; echo rhs=$?
tail -3 gpurun_out/pytest_rhs.log
timeout 300 python tools/profile_step.py --config c5 --steps 3 --timing 2>&1 | tail -8
