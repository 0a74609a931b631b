mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_rom_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/micro_rom.py > gpurun_out/micro_rom.log 2>&1
PICROM_GRAM_NO_TMA=1 PICROM_COMBINE_NO_TMA=1 timeout 600 python tools/micro_rom.py > gpurun_out/micro_rom_notma.log 2>&1
timeout 600 python tools/prof_stage.py > gpurun_out/prof_stage.log 2>&1
timeout 1200 python tools/bench_rom.py --config C3 --steps 3 --warmup 1 > gpurun_out/rom_c3.log 2>&1
echo done
