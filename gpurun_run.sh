mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 20"
timeout 200 $B > gpurun_out/b_tma_default.log 2>&1
PICROM_TMA_CFG=8,2 timeout 200 $B > gpurun_out/b_tma_8_2.log 2>&1
PICROM_TMA_CFG=8,4 timeout 200 $B > gpurun_out/b_tma_8_4.log 2>&1
PICROM_NO_TMA=1 timeout 200 $B > gpurun_out/b_notma_u4b3.log 2>&1
for v in u2_b3 u4_b2 u2_b2; do PICROM_NO_TMA=1 PICROM_LIB=$PWD/build/variants/lib_$v.so timeout 200 $B > gpurun_out/b_notma_$v.log 2>&1; done
PICROM_NO_TMA=1 PICROM_HIST_KB=36 timeout 200 $B > gpurun_out/b_notma_kb36.log 2>&1
timeout 300 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 5 > gpurun_out/b_c5_tma.log 2>&1
PICROM_NO_TMA=1 timeout 300 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 5 > gpurun_out/b_c5_notma.log 2>&1
timeout 300 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 200 > gpurun_out/b_c1.log 2>&1
echo done
