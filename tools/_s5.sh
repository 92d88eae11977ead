mkdir -p gpurun_out/s5
A=build_exp/base/libgsde.so B=build_exp/early/libgsde.so WORKLOADS="vascular" R=2 bash tools/ab.sh > gpurun_out/s5/ab.txt 2>&1
GSDE_LIB_PATH=build_exp/early/libgsde.so timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s5/pytest.txt 2>&1
echo done
