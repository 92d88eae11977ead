mkdir -p gpurun_out/r3k
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r3k/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r3k/pytest_gpu.txt
GSDE_LIB_PATH=build_exp/CD/libgsde.so timeout 600 python tools/lib_equal.py /tmp/eq_a.npz > gpurun_out/r3k/eq.txt 2>&1
GSDE_LIB_PATH=build_exp/PH/libgsde.so timeout 600 python tools/lib_equal.py /tmp/eq_b.npz >> gpurun_out/r3k/eq.txt 2>&1
python tools/lib_equal.py --compare /tmp/eq_a.npz /tmp/eq_b.npz >> gpurun_out/r3k/eq.txt 2>&1
LIBS="build_exp/CD/libgsde.so build_exp/PH/libgsde.so" WORKLOADS="star3 hub64 vascular" R=2 N=4 bash tools/abn.sh > gpurun_out/r3k/ab.txt 2>&1
echo done
