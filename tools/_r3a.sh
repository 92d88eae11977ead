mkdir -p gpurun_out/r3a
LIBS="build_exp/K2/libgsde.so build_exp/S0/libgsde.so" WORKLOADS="star3 star5_trials" R=2 N=4 bash tools/abn.sh > gpurun_out/r3a/ab.txt 2>&1
echo done
