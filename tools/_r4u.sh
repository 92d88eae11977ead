mkdir -p gpurun_out/r4u
nvidia-smi -L > gpurun_out/r4u/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r4u/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r4u/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4u/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r4u/bench.json 2> gpurun_out/r4u/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r4u/bench_ref.json 2> gpurun_out/r4u/bench_ref.err
echo done
