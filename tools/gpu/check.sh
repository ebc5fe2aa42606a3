# parity + smoke + benches (c5 default, c4); arguments: extra pytest selection
mkdir -p gpurun_out
T=${TAG:-x}
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q ${PYSEL} > gpurun_out/pytest_gpu_$T.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu_$T.log
timeout 600 python tools/profile_step.py --config c5 --steps 2 --timing > gpurun_out/step_c5_$T.log 2>&1; echo step5=$?
cat gpurun_out/step_c5_$T.log
timeout 600 python tools/profile_step.py --config c4 --steps 4 --timing > gpurun_out/step_c4_$T.log 2>&1; echo step4=$?
cat gpurun_out/step_c4_$T.log
