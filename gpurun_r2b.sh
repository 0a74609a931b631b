mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_fullorder_gpu.py tests/test_fem_gpu.py tests/test_config_parity_gpu.py -k "not c3 and not c4" -m gpu -q -p no:cacheprovider -x > gpurun_out/r2b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_pytest.log
bash tools/variants.sh u2b3 u2b4 u3b3
