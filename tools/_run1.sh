set -x
mkdir -p gpurun_out/r1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1/smi.txt
nproc >> gpurun_out/r1/smi.txt; lscpu | head -20 >> gpurun_out/r1/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1/smoke.txt 2>&1
A=build_exp/old/libgsde.so B=paper_2512_02175_b200/libgsde.so WORKLOADS="star3 hub64 vascular star5_trials" R=2 timeout 900 bash tools/ab.sh > gpurun_out/r1/ab.txt 2>&1
A=build_exp/old/libgsde.so B=build_exp/zd4/libgsde.so WORKLOADS="star3" R=2 timeout 300 bash tools/ab.sh >> gpurun_out/r1/ab.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r1/pytest_gpu.txt 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1/ref_arm.txt 2>&1
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/r1/bench.txt 2>&1
echo done
