mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_rom_gpu.py -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/prof_rom_step.py > gpurun_out/prof_rom.log 2>&1
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:rom_ --csv --log-file gpurun_out/rom_launches.csv python tools/prof_rom_step.py 1000000 > gpurun_out/ncu_rom.log 2>&1
echo done
