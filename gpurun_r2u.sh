mkdir -p gpurun_out
out=gpurun_out/r2u_steps.log; : > $out
for v in default m8 m8nocl; do
  if [ "$v" = default ]; then lib=""; else lib="PICROM_LIB=paper_2201_05555_b200/variants/libpicrom_$v.so"; fi
  echo "== $v" >> $out
  env $lib timeout 300 python tools/step_timing.py 10 1,2 2>&1 | grep "nx=128 d=3" >> $out
  env $lib timeout 100 python tools/cluster_probe.py 2>&1 | head -2 >> $out
done
