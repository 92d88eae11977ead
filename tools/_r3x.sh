mkdir -p gpurun_out/r3x
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r3x/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r3x/pytest_gpu.txt
LIBS="build_exp/T32/libgsde.so build_exp/SV/libgsde.so" WORKLOADS="star3 hub64 vascular" R=2 N=4 bash tools/abn.sh > gpurun_out/r3x/ab.txt 2>&1
echo done
