mkdir -p gpurun_out/r2g
LIBS="build_exp/v3/libgsde.so build_exp/v5/libgsde.so build_exp/A/libgsde.so build_exp/B/libgsde.so" WORKLOADS="star3 hub64 vascular star5_trials" R=2 N=5 bash tools/abn.sh > gpurun_out/r2g/ab.txt 2>&1
echo done
