mkdir -p gpurun_out/r4j
GSDE_BENCH_SHARED_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r4j/bench2.json 2> gpurun_out/r4j/bench2.err
echo "rc=$?" >> gpurun_out/r4j/bench2.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4j/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r4j/bench.json 2> gpurun_out/r4j/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r4j/bench_ref.json 2> gpurun_out/r4j/bench_ref.err
echo done
