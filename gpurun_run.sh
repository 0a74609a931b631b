mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 50"
for u in 3 6; do PICROM_LIB=$PWD/build/variants/lib_u$u.so timeout 300 $B > gpurun_out/b_u$u.log 2>&1; done
timeout 300 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 20 > gpurun_out/b_c5.log 2>&1
timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/b_c1.log 2>&1
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 10"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"step_kernel" -s 6 -c 1 -o gpurun_out/prof_step $CMD > gpurun_out/ncu_full.log 2>&1
echo done
