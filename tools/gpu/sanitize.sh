#!/bin/bash
# one compute-sanitizer tool per call (B200_PROFILING.md): c1 and c2 steps through the library
TOOL=${1:-memcheck}
mkdir -p gpurun_out
python tools/profile_step.py --config c1 --steps 2 > gpurun_out/san_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool $TOOL --error-exitcode 9 --log-file gpurun_out/san_${TOOL}_c1.log \
    python tools/profile_step.py --config c1 --steps 2 > gpurun_out/san_${TOOL}_c1.out 2>&1; echo c1=$?
timeout 1800 compute-sanitizer --tool $TOOL --error-exitcode 9 --log-file gpurun_out/san_${TOOL}_c2.log \
    python tools/profile_step.py --config c2 --steps 1 > gpurun_out/san_${TOOL}_c2.out 2>&1; echo c2=$?
tail -3 gpurun_out/san_${TOOL}_c1.log gpurun_out/san_${TOOL}_c2.log
