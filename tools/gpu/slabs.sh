# the slab-decomposed bench path on one GPU (torchrun, NCCL world of 1), c4 and c5
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
   bench.py --slabs --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/slabs_c4.json 2> gpurun_out/slabs_c4.err; echo c4=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 \
   bench.py --slabs --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/slabs_c5.json 2> gpurun_out/slabs_c5.err; echo c5=$?
cut -c1-400 gpurun_out/slabs_c4.json; cut -c1-400 gpurun_out/slabs_c5.json; tail -n 5 gpurun_out/slabs_c4.err; tail -n 5 gpurun_out/slabs_c5.err
