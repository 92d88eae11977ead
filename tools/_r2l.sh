mkdir -p gpurun_out/r2l
timeout 900 python bench.py > gpurun_out/r2l/bench.json 2> gpurun_out/r2l/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2l/bench_ref.json 2> gpurun_out/r2l/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2l/launches_star3.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-extras > /dev/null 2>&1
for w in star3; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:native_ensemble_kernel -c 1 \
    -o /tmp/ncu_$w python bench.py --workload $w --steps 1 --warmup 0 --no-extras --no-cpu > gpurun_out/r2l/ncu_$w.log 2>&1
  python tools/ncu_summary.py /tmp/ncu_$w.ncu-rep > gpurun_out/r2l/sum_$w.json 2>&1
  python tools/ncu_lines.py /tmp/ncu_$w.ncu-rep 60 > gpurun_out/r2l/lines_$w.txt 2>&1
done
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t python tools/sanitize.py > gpurun_out/r2l/san_$t.txt 2>&1
done
echo done
