mkdir -p gpurun_out/r3y
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r3y/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r3y/pytest_gpu.txt
LIBS="build_exp/T32/libgsde.so build_exp/TU/libgsde.so" WORKLOADS="star5_trials star3" R=2 N=4 bash tools/abn.sh > gpurun_out/r3y/ab.txt 2>&1
GSDE_LIB_PATH=build_exp/TU/libgsde.so timeout 900 python tools/trials_scale_check.py gpurun_out/r3y/trials_scale.csv > gpurun_out/r3y/trials.txt 2>&1
echo done
