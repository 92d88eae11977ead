mkdir -p gpurun_out/r3e
GSDE_LIB_PATH=build_exp/S0/libgsde.so timeout 600 python tools/lib_equal.py /tmp/eq_a.npz > gpurun_out/r3e/eq.txt 2>&1
GSDE_LIB_PATH=build_exp/CD/libgsde.so timeout 600 python tools/lib_equal.py /tmp/eq_b.npz >> gpurun_out/r3e/eq.txt 2>&1
python tools/lib_equal.py --compare /tmp/eq_a.npz /tmp/eq_b.npz >> gpurun_out/r3e/eq.txt 2>&1
echo done
