# dev: ROM-side validation + timings of the default library and named variants
mkdir -p gpurun_out
out=gpurun_out/exp_rom.log; : > $out
timeout 1200 python -m pytest tests/test_tall_gpu.py tests/test_rom_gpu.py -m gpu -x -q -p no:cacheprovider > gpurun_out/exp_rom_pytest.log 2>&1; echo "pytest rc=$?" >> $out
tail -3 gpurun_out/exp_rom_pytest.log >> $out
for v in default "$@"; do
  if [ "$v" = default ]; then lib=""; else lib="PICROM_LIB=paper_2201_05555_b200/variants/libpicrom_$v.so"; fi
  echo "== $v micro_rom" >> $out
  env $lib timeout 300 python tools/micro_rom.py >> $out 2>&1
done
echo "== window svd pieces" >> $out
timeout 600 python tools/prof_window_svd.py >> $out 2>&1
timeout 900 python -m pytest tests/test_config_parity_gpu.py -m gpu -x -q -p no:cacheprovider -k "c3 or c4 or C3 or C4" > gpurun_out/exp_rom_parity.log 2>&1; echo "parity rc=$?" >> $out
tail -3 gpurun_out/exp_rom_parity.log >> $out
timeout 900 python tools/bench_rom.py --config C4 --steps 5 --warmup 1 > gpurun_out/exp_rom_c4.log 2>&1
tail -1 gpurun_out/exp_rom_c4.log | cut -c1-700 >> $out
timeout 900 python tools/bench_rom.py --config C3 --steps 5 --warmup 2 --no-cpu > gpurun_out/exp_rom_c3.log 2>&1
tail -1 gpurun_out/exp_rom_c3.log | cut -c1-500 >> $out
cat $out
