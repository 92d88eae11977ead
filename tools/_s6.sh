mkdir -p gpurun_out/s6
LIBS="build_exp/base/libgsde.so build_exp/early/libgsde.so build_exp/esm/libgsde.so" WORKLOADS="hub64 vascular" R=2 bash tools/abn.sh > gpurun_out/s6/abn.txt 2>&1
echo done
