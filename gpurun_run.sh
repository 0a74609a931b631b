# Round-end style validation on one B200: GPU tests, smoke, bench (both arms), C5/C1/C4 lines,
# ncu launch list + full captures (exported to CSV on the box; the .ncu-rep files stay there)
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
export_rep() {   # $1 = report stem under gpurun_out/
  $NCU -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/ncu_$1_raw.csv 2>/dev/null
  $NCU -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/ncu_$1_details.csv 2>/dev/null
  $NCU -i gpurun_out/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_$1_sass.csv 2>/dev/null
  rm -f gpurun_out/$1.ncu-rep
}
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
SECONDS=0; timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$? wall=${SECONDS}s" >> gpurun_out/bench_full.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --no-rom > gpurun_out/bench_c5.log 2>&1
timeout 600 python bench.py --config C1 --steps 20 --warmup 3 --no-cpu-baseline --no-rom > gpurun_out/bench_c1.log 2>&1
timeout 1500 python tools/bench_rom.py --config C4 --steps 5 --warmup 1 > gpurun_out/rom_c4.log 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-rom --e2e-steps 2 > gpurun_out/ncu_launch.log 2>&1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:step_kernel -s 5 -c 1 -o gpurun_out/step_c2 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-rom --e2e-steps 2 > gpurun_out/ncu_step.log 2>&1
export_rep step_c2
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:tall_atb_kernel -s 24 -c 1 -o gpurun_out/tall_atb_c4 -f python tools/prof_window_svd.py > gpurun_out/ncu_tall_atb.log 2>&1
export_rep tall_atb_c4
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:wide_combine_kernel -s 3 -c 1 -o gpurun_out/wide_combine6_c4 -f python tools/prof_window_svd.py > gpurun_out/ncu_wide_combine.log 2>&1
export_rep wide_combine6_c4
timeout 300 python tools/micro_rom.py > gpurun_out/micro_rom.log 2>&1
timeout 600 python tools/prof_window_svd.py > gpurun_out/prof_window_svd.log 2>&1
echo done
