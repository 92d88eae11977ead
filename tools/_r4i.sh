mkdir -p gpurun_out/r4i
timeout 600 python -m pytest tests/test_gpu_streamed.py -q -x > gpurun_out/r4i/streamed.txt 2>&1
echo "rc=$?" >> gpurun_out/r4i/streamed.txt
timeout 300 python tools/e2e_star3_probe.py > gpurun_out/r4i/star3_probe.txt 2>&1
GSDE_FORCE_STREAMING=1 timeout 900 python tools/e2e_streamed_ab.py > gpurun_out/r4i/ab.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r4i/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r4i/pytest_gpu.txt
echo done
