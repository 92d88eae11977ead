mkdir -p gpurun_out/r4k
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t python tools/sanitize.py > gpurun_out/r4k/san_$t.txt 2>&1
  echo "$t rc=$?" >> gpurun_out/r4k/san_$t.txt
done
echo done
