mkdir -p gpurun_out/r2d
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2d/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r2d/pytest_gpu.txt
GSDE_LIB_PATH=build_exp/v3/libgsde.so timeout 900 python -m pytest tests -m gpu -q -x -k "lean or parity or state or inject" > gpurun_out/r2d/pytest_v3.txt 2>&1
echo "rc=$?" >> gpurun_out/r2d/pytest_v3.txt
LIBS="build_exp/v1/libgsde.so build_exp/v2/libgsde.so build_exp/v3/libgsde.so" WORKLOADS="star3 hub64 vascular star5_trials" R=2 N=6 bash tools/abn.sh > gpurun_out/r2d/ab.txt 2>&1
echo done
