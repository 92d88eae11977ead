mkdir -p gpurun_out/r3b
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r3b/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r3b/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3b/smoke.txt 2>&1
timeout 1500 python bench.py > gpurun_out/r3b/bench.json 2> gpurun_out/r3b/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r3b/bench_ref.json 2> gpurun_out/r3b/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r3b/launches_star3.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-extras > /dev/null 2>&1
for w in star3 hub64 vascular star5_trials; do
  k=native_ensemble_kernel; [ "$w" = star5_trials ] && k=native_trials_kernel
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 \
    -o /tmp/ncu_$w python bench.py --workload $w --steps 1 --warmup 0 --no-extras --no-cpu > gpurun_out/r3b/ncu_$w.log 2>&1
  python tools/ncu_summary.py /tmp/ncu_$w.ncu-rep > gpurun_out/r3b/sum_$w.json 2>&1
  python tools/ncu_lines.py /tmp/ncu_$w.ncu-rep 60 > gpurun_out/r3b/lines_$w.txt 2>&1
done
echo done
