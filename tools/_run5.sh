mkdir -p gpurun_out/r5
for w in star3 hub64 vascular star5_trials; do timeout 300 python tools/jitter.py $w 6 2>&1 | tail -1; done > gpurun_out/r5/jitter.txt
timeout 1500 python -m pytest tests/test_gpu_state_parity.py tests/test_gpu_c4.py tests/test_gpu_robustness.py -q -s > gpurun_out/r5/state.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r5/pytest_gpu.txt 2>&1
echo done
