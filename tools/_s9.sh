mkdir -p gpurun_out/s9
LIBS="build_exp/cur/libgsde.so build_exp/q16/libgsde.so build_exp/q10/libgsde.so" WORKLOADS="vascular hub64" R=2 N=4 bash tools/abn.sh > gpurun_out/s9/abn.txt 2>&1
echo done
