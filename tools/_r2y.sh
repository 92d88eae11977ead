mkdir -p gpurun_out/r2y
s=$(date +%s)
timeout 1500 python bench.py > gpurun_out/r2y/bench.json 2> gpurun_out/r2y/bench.err
echo "bench rc=$? seconds=$(( $(date +%s) - s ))" >> gpurun_out/r2y/times.txt
s=$(date +%s)
timeout 900 python bench.py --impl reference > gpurun_out/r2y/bench_ref.json 2> gpurun_out/r2y/bench_ref.err
echo "ref rc=$? seconds=$(( $(date +%s) - s ))" >> gpurun_out/r2y/times.txt
s=$(date +%s)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2y/smoke.txt 2>&1
echo "smoke rc=$? seconds=$(( $(date +%s) - s ))" >> gpurun_out/r2y/times.txt
echo done
