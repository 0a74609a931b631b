# usage: bash tools/exp_step.sh VARIANT...  -- step timing (C2 + two more shapes, C5) of the
# default library and the named variants; runs the FOM GPU tests on the default first
mkdir -p gpurun_out
out=gpurun_out/exp_step.log; : > $out
timeout 900 python -m pytest tests/test_fullorder_gpu.py tests/test_memory_safety_gpu.py tests/test_fem_gpu.py -m gpu -x -q -p no:cacheprovider > gpurun_out/exp_step_pytest.log 2>&1; echo "pytest rc=$?" >> $out
for rep in 1 2; do
for v in default "$@"; do
  if [ "$v" = default ]; then lib=""; else lib="PICROM_LIB=paper_2201_05555_b200/variants/libpicrom_$v.so"; fi
  echo "== $v" >> $out
  env $lib timeout 300 python tools/step_timing.py 20 1,2 0,4,5 >> $out 2>&1
done
done
for v in default "$@"; do
  if [ "$v" = default ]; then lib=""; else lib="PICROM_LIB=paper_2201_05555_b200/variants/libpicrom_$v.so"; fi
  echo "== $v C5" >> $out
  env $lib timeout 300 python tools/step_timing.py 5 1 2 >> $out 2>&1
done
cat $out; tail -5 gpurun_out/exp_step_pytest.log
