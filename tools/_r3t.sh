mkdir -p gpurun_out/r3t
timeout 900 python -m pytest tests/test_fvm.py -m gpu -q > gpurun_out/r3t/pytest_fvm.txt 2>&1
echo "rc=$?" >> gpurun_out/r3t/pytest_fvm.txt
LIBS="build_exp/PDL0/libgsde.so build_exp/PDL2/libgsde.so" WORKLOADS="fvm" R=2 N=4 bash tools/abn.sh > gpurun_out/r3t/ab.txt 2>&1
echo done
