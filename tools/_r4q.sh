mkdir -p gpurun_out/r4q
LIBS="build_exp/B0/libgsde.so build_exp/SU/libgsde.so" WORKLOADS="star3" R=3 N=4 bash tools/abn.sh > gpurun_out/r4q/ab.txt 2>&1
for L in B0 SU; do echo "== $L" >> gpurun_out/r4q/probe.txt; GSDE_LIB_PATH=build_exp/$L/libgsde.so timeout 300 python tools/e2e_star3_probe.py >> gpurun_out/r4q/probe.txt 2>&1; done
echo done
