mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_fullorder_gpu.py tests/test_fem_gpu.py -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
B="python bench.py --no-cpu-baseline --e2e-steps 50 --steps 30"
timeout 400 $B > gpurun_out/b_fused.log 2>&1
PICROM_NOSOLVE=1 timeout 400 $B > gpurun_out/b_nosolve.log 2>&1
echo done
