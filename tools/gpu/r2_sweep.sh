#!/bin/bash
# TMA-staged sweeps: parity, then c5 bench with and without them
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tma or sweeps or c1_full or c4_full or derivative or c2_shape" > gpurun_out/pytest_sweep.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_sweep.log
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tma.json 2> gpurun_out/bench_tma.err; echo bench=$?
ADI_SW_TMA=0 timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/bench_legacy.json 2> gpurun_out/bench_legacy.err; echo bench_legacy=$?
python - <<'PY'
import json
for f in ("gpurun_out/bench_tma.json", "gpurun_out/bench_legacy.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "no json", e); continue
    print(f, "ms/step %.2f" % d["ms_per_step"], {k: (round(v["ms_total"] / v["launches"], 3), round(v.get("frac", 0), 3)) for k, v in d["kernels"].items()})
PY
tail -3 gpurun_out/bench_tma.err
