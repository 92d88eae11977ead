mkdir -p gpurun_out/r2j
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2j/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r2j/pytest_gpu.txt
LIBS="build_exp/v6/libgsde.so build_exp/v7np/libgsde.so build_exp/v7/libgsde.so" WORKLOADS="star3 hub64 vascular star5_trials" R=2 N=5 bash tools/abn.sh > gpurun_out/r2j/ab.txt 2>&1
echo done
