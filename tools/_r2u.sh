mkdir -p gpurun_out/r2u
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2u/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r2u/pytest_gpu.txt
for lib in build_exp/cur/libgsde.so build_exp/P1/libgsde.so; do
  echo "== $lib" >> gpurun_out/r2u/e2e.txt
  GSDE_LIB_PATH=$lib timeout 600 python tools/e2e_time.py star3 hub64 vascular >> gpurun_out/r2u/e2e.txt 2>&1
done
LIBS="build_exp/cur/libgsde.so build_exp/P1/libgsde.so" WORKLOADS="star3 hub64 vascular" R=1 N=4 bash tools/abn.sh > gpurun_out/r2u/ab.txt 2>&1
echo done
