mkdir -p gpurun_out/r2c
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t python tools/sanitize.py > gpurun_out/r2c/san_$t.txt 2>&1
  echo "$t rc=$?" >> gpurun_out/r2c/san_$t.txt
done
GSDE_FORCE_GLOBAL_BINS=1 GSDE_CHUNK_PARTICLES=7777 timeout 900 compute-sanitizer --tool memcheck python tools/sanitize.py > gpurun_out/r2c/san_memcheck_globalbins_chunked.txt 2>&1
echo "rc=$?" >> gpurun_out/r2c/san_memcheck_globalbins_chunked.txt
echo done
