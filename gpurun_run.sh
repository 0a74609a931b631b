mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/variants.log
for c in C2 C5 C1; do
  echo "== main $c" >> gpurun_out/variants.log
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-rom --e2e-steps 2 2>&1 | tee -a gpurun_out/variants_raw.log | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step'], d['roofline']['frac'])" >> gpurun_out/variants.log 2>&1
done
echo done
