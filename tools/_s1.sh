mkdir -p gpurun_out/s1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s1/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s1/smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s1/pytest_gpu.txt 2>&1
timeout 600 python bench.py > gpurun_out/s1/bench.json 2> gpurun_out/s1/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/s1/bench_ref.json 2> gpurun_out/s1/bench_ref.err
echo done
