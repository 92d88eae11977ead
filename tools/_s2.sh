mkdir -p gpurun_out/s2
A=build_exp/base/libgsde.so B=build_exp/res/libgsde.so WORKLOADS="vascular hub64" R=2 bash tools/ab.sh > gpurun_out/s2/ab.txt 2>&1
echo done
