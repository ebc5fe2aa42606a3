mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ov1.json 2>&1; echo b1=$?
ADI_OVERLAP=0 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ov0.json 2>&1; echo b0=$?
python -c "
import json
for f in ['gpurun_out/bench_ov1.json','gpurun_out/bench_ov0.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['ms_per_step'], d['value'])"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ov.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_ov.log
