mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_rom_gpu.py -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/prof_rom_step.py > gpurun_out/prof_rom.log 2>&1
timeout 900 python tools/bench_rom.py --config C3 --steps 5 --warmup 2 > gpurun_out/rom_c3.log 2>&1; echo "rc=$?" >> gpurun_out/rom_c3.log
echo done
