mkdir -p gpurun_out/r2z
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2z/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r2z/pytest_gpu.txt
LIBS="build_exp/K2/libgsde.so build_exp/SN/libgsde.so" WORKLOADS="star3 star5_trials" R=2 N=4 bash tools/abn.sh > gpurun_out/r2z/ab.txt 2>&1
for lib in build_exp/K2/libgsde.so build_exp/SN/libgsde.so; do
  echo "== $lib" >> gpurun_out/r2z/e2e.txt
  GSDE_LIB_PATH=$lib timeout 600 python tools/e2e_time.py star3 >> gpurun_out/r2z/e2e.txt 2>&1
done
echo done
