mkdir -p gpurun_out/r4f
timeout 600 python -m pytest tests/test_gpu_streamed.py -q -x > gpurun_out/r4f/streamed.txt 2>&1
echo "rc=$?" >> gpurun_out/r4f/streamed.txt
timeout 900 python tools/e2e_streamed_ab.py vascular > gpurun_out/r4f/ab.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r4f/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r4f/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4f/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r4f/bench.json 2> gpurun_out/r4f/bench.err
echo done
