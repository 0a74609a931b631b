mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 python bench.py --steps 20 --warmup 5 --no-rom --no-cpu-baseline > gpurun_out/r2ab_bench.log 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2ab_launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-rom --e2e-steps 16 > gpurun_out/r2ab_ncu_launch.log 2>&1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:step_kernel -s 12 -c 2 -o gpurun_out/r2ab_step_c2 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-rom --e2e-steps 16 > gpurun_out/r2ab_ncu_step.log 2>&1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:step_kernel -s 6 -c 1 -o gpurun_out/r2ab_step_c5 -f python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-rom --e2e-steps 4 > gpurun_out/r2ab_ncu_c5.log 2>&1
echo done
