mkdir -p gpurun_out/r2v
GSDE_BENCH_SHARED_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r2v/bench2.json 2> gpurun_out/r2v/bench2.err
echo "rc=$?" >> gpurun_out/r2v/bench2.err
GSDE_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/r2v/ref2.json 2> gpurun_out/r2v/ref2.err
echo "rc=$?" >> gpurun_out/r2v/ref2.err
echo done
