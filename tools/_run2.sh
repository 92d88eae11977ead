set -x
mkdir -p gpurun_out/r2
A=build_exp/old/libgsde.so B=paper_2512_02175_b200/libgsde.so WORKLOADS="star3 hub64 vascular star5_trials" R=1 timeout 900 bash tools/ab.sh > gpurun_out/r2/ab.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2/pytest_gpu.txt 2>&1
SECONDS=0; timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r2/bench.txt 2>&1; echo "bench_s $SECONDS" >> gpurun_out/r2/bench.txt
echo done
