# ncu --set full of the manifold-map kernels inside a C3 step (gram_mma, wide_combine<3>), CSV export
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for k in gram_mma_kernel wide_combine_kernel; do
  timeout 1200 $NCU --set full --import-source on --clock-control none -k regex:$k -s 12 -c 1 -o gpurun_out/c3_$k -f python tools/bench_rom.py --config C3 --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_c3_$k.log 2>&1
  $NCU -i gpurun_out/c3_$k.ncu-rep --page raw --csv > gpurun_out/ncu_c3_${k}_raw.csv 2>/dev/null
  $NCU -i gpurun_out/c3_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_c3_${k}_sass.csv 2>/dev/null
  rm -f gpurun_out/c3_$k.ncu-rep
done
echo done
