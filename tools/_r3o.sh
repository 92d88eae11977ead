mkdir -p gpurun_out/r3o
timeout 600 python tools/c5_shard_times.py > gpurun_out/r3o/c5.txt 2>&1
echo done
