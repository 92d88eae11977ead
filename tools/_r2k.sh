mkdir -p gpurun_out/r2k
LIBS="build_exp/v7c/libgsde.so build_exp/q10s2/libgsde.so build_exp/q12s3/libgsde.so build_exp/q12s4/libgsde.so build_exp/q16s4/libgsde.so build_exp/q18s3/libgsde.so" WORKLOADS="hub64 vascular" R=2 N=4 bash tools/abn.sh > gpurun_out/r2k/ab.txt 2>&1
echo done
