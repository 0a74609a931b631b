mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_rom_gpu.py tests/test_config_parity_gpu.py -k "deim or hyper or c4" -m gpu -q -p no:cacheprovider > gpurun_out/r2l_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_pytest.log
timeout 300 python tools/prof_deim.py > gpurun_out/r2l_prof_deim.log 2>&1
