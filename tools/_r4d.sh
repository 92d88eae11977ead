mkdir -p gpurun_out/r4d
timeout 600 python -m pytest tests/test_gpu_streamed.py -q -x > gpurun_out/r4d/streamed.txt 2>&1
echo "rc=$?" >> gpurun_out/r4d/streamed.txt
timeout 900 python tools/e2e_streamed_ab.py > gpurun_out/r4d/ab.txt 2>&1
echo done
