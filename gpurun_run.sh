mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/variants.log
for v in "pdl X=1" "nopdl PICROM_NO_PDL=1"; do
  set -- $v; name=$1; shift
  for c in C2 C1; do
    echo "== $name $c" >> gpurun_out/variants.log
    env "$@" timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-rom 2>&1 | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step'], d['roofline']['frac'], 'e2e', d['e2e']['value']/1e9, d['e2e']['seconds'])" >> gpurun_out/variants.log 2>&1
  done
done
echo done
