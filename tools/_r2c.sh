mkdir -p gpurun_out/r2c
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2c/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r2c/pytest_gpu.txt
A=build_exp/base/libgsde.so B=build_exp/v1/libgsde.so WORKLOADS="star3 hub64 vascular" R=2 N=6 bash tools/ab.sh > gpurun_out/r2c/ab.txt 2>&1
echo done
