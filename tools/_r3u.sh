mkdir -p gpurun_out/r3u
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r3u/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r3u/pytest_gpu.txt
LIBS="build_exp/CD/libgsde.so build_exp/UNI/libgsde.so" WORKLOADS="hub64 vascular" R=2 N=4 bash tools/abn.sh > gpurun_out/r3u/ab.txt 2>&1
echo done
