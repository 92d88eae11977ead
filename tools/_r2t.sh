mkdir -p gpurun_out/r2t
LIBS="build_exp/cur/libgsde.so build_exp/T1/libgsde.so" WORKLOADS="star5_trials" R=3 N=4 bash tools/abn.sh > gpurun_out/r2t/ab.txt 2>&1
echo done
