mkdir -p gpurun_out/r3i
TABLES_ONLY=3 timeout 900 python tools/paper_tables.py gpurun_out/r3i > gpurun_out/r3i/t3.txt 2>&1
TABLES_ONLY=4 timeout 1500 python tools/paper_tables.py gpurun_out/r3i > gpurun_out/r3i/t4.txt 2>&1
echo done
