mkdir -p gpurun_out
out=gpurun_out/exp_rom3.log; : > $out
timeout 1200 python -m pytest tests/test_tall_gpu.py tests/test_rom_gpu.py -m gpu -x -q -p no:cacheprovider > gpurun_out/exp_rom3_pytest.log 2>&1; echo "pytest rc=$?" >> $out
tail -3 gpurun_out/exp_rom3_pytest.log >> $out
timeout 900 python tools/bench_rom.py --config C4 --steps 5 --warmup 1 > gpurun_out/exp_rom3_c4.log 2>&1
tail -1 gpurun_out/exp_rom3_c4.log | cut -c1-700 >> $out
timeout 600 python tools/prof_rom_kernels.py C4 > gpurun_out/prof_kernels_C4_step.txt 2>&1
timeout 600 python tools/prof_rom_host.py C4 5 > gpurun_out/prof_host_C4_step.txt 2>&1
head -24 gpurun_out/prof_kernels_C4_step.txt | cut -c1-150 >> $out
tail -24 gpurun_out/prof_host_C4_step.txt >> $out
cat $out
