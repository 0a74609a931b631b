mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --no-rom > gpurun_out/bench_c5.log 2>&1
timeout 600 python bench.py --config C1 --steps 20 --warmup 3 --no-cpu-baseline --no-rom > gpurun_out/bench_c1.log 2>&1
timeout 1500 python tools/bench_rom.py --config C4 --steps 5 --warmup 1 > gpurun_out/rom_c4.log 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-rom --e2e-steps 2 > gpurun_out/ncu_launch.log 2>&1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:step_kernel -s 5 -c 1 -o gpurun_out/step_c2 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-rom --e2e-steps 2 > gpurun_out/ncu_step.log 2>&1
echo done
