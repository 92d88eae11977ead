mkdir -p gpurun_out/r3s
timeout 900 python -m pytest tests/test_fvm.py tests/test_fvm_pack.py -m gpu -q > gpurun_out/r3s/pytest_fvm.txt 2>&1
echo "rc=$?" >> gpurun_out/r3s/pytest_fvm.txt
LIBS="build_exp/PDL0/libgsde.so build_exp/PDL1/libgsde.so" WORKLOADS="fvm" R=2 N=4 bash tools/abn.sh > gpurun_out/r3s/ab.txt 2>&1
GSDE_LIB_PATH=build_exp/PDL1/libgsde.so timeout 600 python tools/fvm_small_rate.py > gpurun_out/r3s/small.txt 2>&1
echo done
