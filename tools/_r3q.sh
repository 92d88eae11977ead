mkdir -p gpurun_out/r3q
rm -rf /tmp/gsde_numba_cache
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r3q/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r3q/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3q/smoke.txt 2>&1
s=$(date +%s); timeout 1500 python bench.py > gpurun_out/r3q/bench.json 2> gpurun_out/r3q/bench.err; echo "bench rc=$? s=$(( $(date +%s) - s ))" >> gpurun_out/r3q/times.txt
s=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/r3q/bench_ref.json 2> gpurun_out/r3q/bench_ref.err; echo "ref rc=$? s=$(( $(date +%s) - s ))" >> gpurun_out/r3q/times.txt
echo done
