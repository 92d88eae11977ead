mkdir -p gpurun_out/r2e
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2e/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r2e/pytest_gpu.txt
timeout 300 python tools/carry_check.py /tmp/c_prod.npz > gpurun_out/r2e/carry.txt 2>&1
GSDE_LIB_PATH=build_exp/carry/libgsde.so timeout 600 python tools/carry_check.py /tmp/c_carry.npz >> gpurun_out/r2e/carry.txt 2>&1
python tools/carry_check.py --compare /tmp/c_prod.npz /tmp/c_carry.npz >> gpurun_out/r2e/carry.txt 2>&1
LIBS="build_exp/v3/libgsde.so build_exp/v4/libgsde.so" WORKLOADS="star3 hub64 vascular star5_trials" R=2 N=6 bash tools/abn.sh > gpurun_out/r2e/ab.txt 2>&1
echo done
