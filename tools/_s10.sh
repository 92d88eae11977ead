mkdir -p gpurun_out/s10
LIBS="build_exp/cur/libgsde.so build_exp/qrec/libgsde.so" WORKLOADS="vascular" R=2 N=5 bash tools/abn.sh > gpurun_out/s10/abn.txt 2>&1
GSDE_LIB_PATH=build_exp/qrec/libgsde.so timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s10/pytest.txt 2>&1
echo done
