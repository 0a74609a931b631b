mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fullorder_gpu.py tests/test_fem_gpu.py -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/variants.log
for rep in 1 2; do
for c in C2 C5 C1; do
  echo "== main $c" >> gpurun_out/variants.log
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-rom 2>&1 | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step'], d['roofline']['frac'], d['e2e']['value']/1e9)" >> gpurun_out/variants.log 2>&1
done
done
echo done
