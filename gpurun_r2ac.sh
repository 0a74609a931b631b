mkdir -p gpurun_out
out=gpurun_out/r2ac_steps.log; : > $out
for v in default u4m3 u5m2 u3m3; do
  if [ "$v" = default ]; then lib=""; else lib="PICROM_LIB=paper_2201_05555_b200/variants/libpicrom_$v.so"; fi
  echo "== $v" >> $out
  env $lib timeout 300 python tools/step_timing.py 10 1,2 2>&1 | grep -E "nx=128 d=3|nx=64" >> $out
done
