mkdir -p gpurun_out/r2w
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2w/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r2w/pytest_gpu.txt
LIBS="build_exp/P1/libgsde.so build_exp/K1/libgsde.so" WORKLOADS="star5_trials star3" R=2 N=4 bash tools/abn.sh > gpurun_out/r2w/ab.txt 2>&1
echo done
