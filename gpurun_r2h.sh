mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not c3_ and not c4_" > gpurun_out/r2h_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_smoke.log
timeout 600 python bench.py --no-rom > gpurun_out/r2h_bench.log 2>&1
timeout 600 python bench.py --config C5 --steps 5 --no-rom --no-cpu-baseline > gpurun_out/r2h_bench_c5.log 2>&1
timeout 300 python bench.py --config C1 --steps 50 --no-rom --no-cpu-baseline > gpurun_out/r2h_bench_c1.log 2>&1
