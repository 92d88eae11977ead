mkdir -p gpurun_out/s3
A=build_exp/base/libgsde.so B=build_exp/grp/libgsde.so WORKLOADS="star5_trials" R=2 bash tools/ab.sh > gpurun_out/s3/ab.txt 2>&1
GSDE_LIB_PATH=build_exp/grp/libgsde.so timeout 900 python -m pytest tests -m gpu -q -x -k "trial or exit or distributed or shard" > gpurun_out/s3/pytest_trials.txt 2>&1
echo done
