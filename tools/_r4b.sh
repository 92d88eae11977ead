mkdir -p gpurun_out/r4b
timeout 600 python -m pytest tests/test_gpu_streamed.py -q -x > gpurun_out/r4b/streamed.txt 2>&1
echo "rc=$?" >> gpurun_out/r4b/streamed.txt
timeout 300 python tools/e2e_star3_probe.py > gpurun_out/r4b/star3_probe.txt 2>&1
timeout 900 python tools/e2e_streamed_ab.py > gpurun_out/r4b/ab.txt 2>&1
echo done
