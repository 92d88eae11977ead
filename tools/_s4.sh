mkdir -p gpurun_out/s4
for v in grp; do
GSDE_LIB_PATH=build_exp/$v/libgsde.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:native_trials_kernel -c 1 \
    -o gpurun_out/s4/$v python bench.py --workload star5_trials --steps 1 --warmup 0 --no-extras --no-cpu > gpurun_out/s4/$v.log 2>&1
echo $v $?
done
for v in grp; do
python tools/ncu_summary.py gpurun_out/s4/$v.ncu-rep > gpurun_out/s4/$v.sum.txt 2>&1
python tools/ncu_lines.py gpurun_out/s4/$v.ncu-rep 30 > gpurun_out/s4/$v.lines.txt 2>&1
ls -la gpurun_out/s4/$v.ncu-rep >> gpurun_out/s4/sizes.txt
rm -f gpurun_out/s4/$v.ncu-rep
done
