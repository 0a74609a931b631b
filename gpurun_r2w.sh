mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_rom_gpu.py tests/test_config_parity_gpu.py tests/test_parallel_rom_gpu.py tests/test_memory_safety_gpu.py -k "not c2_ and not c1_ and not c5_" -m gpu -q -p no:cacheprovider > gpurun_out/r2w_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2w_pytest.log
timeout 600 python tools/bench_rom.py --config C3 --no-cpu > gpurun_out/r2w_c3.log 2>&1
timeout 600 python tools/bench_rom.py --config C4 --no-cpu > gpurun_out/r2w_c4.log 2>&1
