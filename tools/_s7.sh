mkdir -p gpurun_out/s7
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s7/smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s7/pytest_gpu.txt 2>&1
timeout 600 python bench.py > gpurun_out/s7/bench.json 2> gpurun_out/s7/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/s7/bench_ref.json 2> gpurun_out/s7/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s7/launches.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu > gpurun_out/s7/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:native_ensemble_kernel -c 1 -o gpurun_out/s7/vascular python bench.py --workload vascular --steps 1 --warmup 0 --no-extras --no-cpu > gpurun_out/s7/vascular.log 2>&1
python tools/ncu_summary.py gpurun_out/s7/vascular.ncu-rep > gpurun_out/s7/vascular.sum.txt 2>&1
python tools/ncu_lines.py gpurun_out/s7/vascular.ncu-rep 60 > gpurun_out/s7/vascular.lines.txt 2>&1
ncu -i gpurun_out/s7/vascular.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum > gpurun_out/s7/vascular.dram.csv 2>&1
rm -f gpurun_out/s7/vascular.ncu-rep
echo done
