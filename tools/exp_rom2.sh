mkdir -p gpurun_out
out=gpurun_out/exp_rom2.log; : > $out
timeout 1200 python -m pytest tests/test_tall_gpu.py tests/test_rom_gpu.py tests/test_memory_safety_gpu.py -m gpu -x -q -p no:cacheprovider > gpurun_out/exp_rom2_pytest.log 2>&1; echo "pytest rc=$?" >> $out
tail -3 gpurun_out/exp_rom2_pytest.log >> $out
timeout 900 python -m pytest tests/test_config_parity_gpu.py -m gpu -x -q -p no:cacheprovider -k "c3 or c4 or C3 or C4" > gpurun_out/exp_rom2_parity.log 2>&1; echo "parity rc=$?" >> $out
tail -3 gpurun_out/exp_rom2_parity.log >> $out
timeout 900 python tools/bench_rom.py --config C4 --steps 5 --warmup 1 > gpurun_out/exp_rom2_c4.log 2>&1
tail -1 gpurun_out/exp_rom2_c4.log | cut -c1-700 >> $out
timeout 600 python tools/prof_rom_kernels.py C4 > gpurun_out/exp_rom2_kern_c4.log 2>&1
head -30 gpurun_out/exp_rom2_kern_c4.log | cut -c1-150 >> $out
cat $out
