# c4 golden (500 oracle steps at 128^3, host cores of the GPU box; resumes build/golden_ckpt/c4.npz)
# while the GPU profiles the TMA sweeps and times the tuning variants
mkdir -p gpurun_out
ORC_THREADS=${ORC_THREADS:-14} nohup python tools/make_golden.py c4 > gpurun_out/make_golden_c4.log 2>&1 &
GP=$!
bash tools/gpu/r2_prof_mass.sh > gpurun_out/prof_mass.log 2>&1
bash tools/gpu/variants3.sh > gpurun_out/variants_r2d.log 2>&1
cat gpurun_out/variants_r2d.log
wait $GP
cp tests/golden/c4_golden.npz gpurun_out/ 2>/dev/null
tail -3 gpurun_out/make_golden_c4.log
