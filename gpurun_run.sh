mkdir -p gpurun_out
: > gpurun_out/variants.log
for cfg in "main X=1" "u8 PICROM_LIB=paper_2201_05555_b200/variants/libpicrom_u8.so" "tma PICROM_TMA=1" "u8hist40 PICROM_LIB=paper_2201_05555_b200/variants/libpicrom_u8.so PICROM_HIST_KB=40"; do
  set -- $cfg; name=$1; shift
  for c in C2 C5 C1; do
    echo "== $name $c" >> gpurun_out/variants.log
    env "$@" timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-rom --e2e-steps 2 2>&1 | tee -a gpurun_out/variants_raw.log | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step'], d['roofline']['frac'])" >> gpurun_out/variants.log 2>&1
  done
done
echo done
