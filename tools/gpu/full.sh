#!/bin/bash
# full GPU suite, smoke, default bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
print("ms/step %.2f value %.3e e2e %.3e" % (d["ms_per_step"], d["value"], d["e2e"]["value"]), "roofline", d["roofline"]["kernel"], round(d["roofline"]["frac"], 3), "step_frac", round(d["step_hbm_frac"], 3))
print({k: (round(v["ms_total"] / v["launches"], 3), round(v.get("frac", 0), 3)) for k, v in d["kernels"].items()}, d["clocks"], d["parity"])
PY
