mkdir -p gpurun_out
timeout 400 python tools/step_timing.py 10 1,2,4 > gpurun_out/r2d_steps.log 2>&1
timeout 900 python -m pytest tests/test_fullorder_gpu.py tests/test_fem_gpu.py tests/test_config_parity_gpu.py -k "not c3 and not c4" -m gpu -q -p no:cacheprovider > gpurun_out/r2d_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_pytest.log
timeout 600 python bench.py --no-rom --no-cpu-baseline > gpurun_out/r2d_bench.log 2>&1
timeout 600 python bench.py --config C5 --steps 5 --no-rom --no-cpu-baseline > gpurun_out/r2d_bench_c5.log 2>&1
