mkdir -p gpurun_out/s8
for t in memcheck initcheck racecheck synccheck; do
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py > gpurun_out/s8/r02_v15_$t.txt 2>&1
  echo "$t rc=$?" >> gpurun_out/s8/r02_v15_$t.txt
done
echo done
