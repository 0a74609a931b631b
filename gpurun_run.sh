mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fullorder_gpu.py tests/test_fem_gpu.py -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-rom > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --no-rom > gpurun_out/bench_c5.log 2>&1
echo done
