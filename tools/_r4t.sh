mkdir -p gpurun_out/r4t
LIBS="build_exp/B0/libgsde.so build_exp/Q12S3/libgsde.so build_exp/Q18S3/libgsde.so build_exp/Q16S4/libgsde.so" WORKLOADS="vascular hub64" R=2 N=4 bash tools/abn.sh > gpurun_out/r4t/ab.txt 2>&1
echo done
