mkdir -p gpurun_out/r4a
timeout 600 python -m pytest tests/test_gpu_streamed.py -q -x > gpurun_out/r4a/streamed.txt 2>&1
echo "rc=$?" >> gpurun_out/r4a/streamed.txt
timeout 300 python tools/e2e_star3_probe.py > gpurun_out/r4a/star3_probe.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r4a/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r4a/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/r4a/bench.json 2> gpurun_out/r4a/bench.err
echo done
