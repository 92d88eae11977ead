mkdir -p gpurun_out/r2x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2x/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r2x/pytest_gpu.txt
LIBS="build_exp/K1/libgsde.so build_exp/K2/libgsde.so" WORKLOADS="star5_trials" R=2 N=4 bash tools/abn.sh > gpurun_out/r2x/ab.txt 2>&1
/usr/bin/time -v timeout 1200 python bench.py > gpurun_out/r2x/bench.json 2> gpurun_out/r2x/bench.err
echo done
