mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_rom_gpu.py -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/prof_deim.py > gpurun_out/prof_deim.log 2>&1
timeout 1500 python tools/bench_rom.py --config C4 --steps 5 --warmup 1 > gpurun_out/rom_c4.log 2>&1; echo "rc=$?" >> gpurun_out/rom_c4.log
echo done
