mkdir -p gpurun_out/r3r
timeout 900 python -m pytest tests/test_fvm.py -m gpu -q > gpurun_out/r3r/pytest_fvm.txt 2>&1
echo "rc=$?" >> gpurun_out/r3r/pytest_fvm.txt
timeout 1200 python bench.py --no-cpu > gpurun_out/r3r/bench.json 2> gpurun_out/r3r/bench.err
echo done
