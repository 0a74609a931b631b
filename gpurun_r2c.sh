mkdir -p gpurun_out
out=gpurun_out/r2c_steps.log; : > $out
for v in default nofix u6b1 nt128u6b3 nt128u4b4; do
  if [ "$v" = default ]; then lib=""; else lib="PICROM_LIB=paper_2201_05555_b200/variants/libpicrom_$v.so"; fi
  echo "== $v" >> $out
  env $lib timeout 300 python tools/step_timing.py 10 >> $out 2>&1
done
timeout 300 python -m pytest tests/test_fullorder_gpu.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2c_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_pytest.log
