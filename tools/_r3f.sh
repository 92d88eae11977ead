mkdir -p gpurun_out/r3f
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r3f/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r3f/pytest_gpu.txt
LIBS="build_exp/CD/libgsde.so build_exp/LD/libgsde.so" WORKLOADS="hub64 vascular" R=2 N=4 bash tools/abn.sh > gpurun_out/r3f/ab.txt 2>&1
echo done
