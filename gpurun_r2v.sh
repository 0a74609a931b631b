mkdir -p gpurun_out
out=gpurun_out/r2v_steps.log; : > $out
for v in m16 default; do
  if [ "$v" = default ]; then lib=""; else lib="PICROM_LIB=paper_2201_05555_b200/variants/libpicrom_$v.so"; fi
  echo "== $v" >> $out
  env $lib timeout 300 python tools/step_timing.py 10 1,2,3,4 2>&1 | grep -E "nx=128 d=3|nx=512 d=3" >> $out
done
