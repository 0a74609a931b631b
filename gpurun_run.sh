mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tall_gpu.py tests/test_rom_gpu.py -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:wide_combine --csv --log-file gpurun_out/wide.csv python tools/prof_rom_step.py 1000000 > gpurun_out/ncu_wide.log 2>&1
timeout 600 python tools/prof_rom_step.py > gpurun_out/prof_rom.log 2>&1
echo done
