mkdir -p gpurun_out/r2s
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2s/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r2s/pytest_gpu.txt
LIBS="build_exp/cur/libgsde.so build_exp/L/libgsde.so" WORKLOADS="star3 hub64 vascular star5_trials" R=2 N=4 bash tools/abn.sh > gpurun_out/r2s/ab.txt 2>&1
echo done
