mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rom_launches.csv python tools/prof_rom_step.py 1000000 > gpurun_out/ncu_rom.log 2>&1
timeout 600 python tools/prof_rom_step.py > gpurun_out/prof_rom.log 2>&1
timeout 1200 python tools/bench_rom.py --config C3 --steps 3 --warmup 1 > gpurun_out/rom_c3.log 2>&1; echo "rc=$?" >> gpurun_out/rom_c3.log
echo done
