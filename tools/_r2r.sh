mkdir -p gpurun_out/r2r
LIBS="build_exp/cur/libgsde.so build_exp/mb5/libgsde.so" WORKLOADS="hub64 vascular" R=2 N=4 bash tools/abn.sh > gpurun_out/r2r/ab.txt 2>&1
echo done
