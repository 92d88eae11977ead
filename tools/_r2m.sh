mkdir -p gpurun_out/r2m
LIBS="build_exp/v7d/libgsde.so build_exp/sb4/libgsde.so" WORKLOADS="star3 star3_ref" R=2 N=5 bash tools/abn.sh > gpurun_out/r2m/ab.txt 2>&1
echo done
