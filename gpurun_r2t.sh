mkdir -p gpurun_out
out=gpurun_out/r2t_steps.log; : > $out
for v in default nocl; do
  if [ "$v" = default ]; then lib=""; else lib="PICROM_LIB=paper_2201_05555_b200/variants/libpicrom_$v.so"; fi
  echo "== $v" >> $out
  env $lib timeout 300 python tools/step_timing.py 10 1,2 >> $out 2>&1
done
PICROM_LIB=paper_2201_05555_b200/variants/libpicrom_tl.so timeout 120 python tools/timeline.py 1 > gpurun_out/r2t_tl.log 2>&1
PICROM_LIB=paper_2201_05555_b200/variants/libpicrom_tl.so timeout 120 python tools/timeline.py 2 >> gpurun_out/r2t_tl.log 2>&1
timeout 900 python -m pytest tests/test_fullorder_gpu.py tests/test_memory_safety_gpu.py tests/test_config_parity_gpu.py -k "not c3 and not c4" -m gpu -q -p no:cacheprovider > gpurun_out/r2t_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_pytest.log
