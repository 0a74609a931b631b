mkdir -p gpurun_out
: > gpurun_out/variants.log
for ms in 2048 512 1024 4096 8192; do
  for c in C1; do
    echo "== minseg $ms $c" >> gpurun_out/variants.log
    PICROM_MIN_SEG=$ms timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-rom --e2e-steps 200 2>&1 | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step'], d['e2e']['value']/1e9)" >> gpurun_out/variants.log 2>&1
  done
done
echo done
