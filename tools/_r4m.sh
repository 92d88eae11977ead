mkdir -p gpurun_out/r4m
LIBS="build_exp/T0/libgsde.so build_exp/TI/libgsde.so" WORKLOADS="star5_trials" R=3 N=4 bash tools/abn.sh > gpurun_out/r4m/ab.txt 2>&1
GSDE_LIB_PATH=build_exp/TI/libgsde.so timeout 900 python -m pytest tests -m gpu -q -x -k "trial or exit or smoke or parity" > gpurun_out/r4m/pytest.txt 2>&1
echo "rc=$?" >> gpurun_out/r4m/pytest.txt
echo done
