# variants timing + the default bench (c5) + c4 bench + reference arm
mkdir -p gpurun_out
T=${TAG:-x}
bash tools/gpu/variants.sh > gpurun_out/variants_$T.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c5_$T.json 2> gpurun_out/bench_c5_$T.err; echo bench5=$?
timeout 600 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_$T.json 2> gpurun_out/bench_c4_$T.err; echo bench4=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err; echo ref=$?
cat gpurun_out/variants_$T.log; cat gpurun_out/bench_c5_$T.json; echo; cat gpurun_out/bench_c4_$T.json; echo; cat gpurun_out/bench_ref_$T.json; tail -3 gpurun_out/bench_c5_$T.err
