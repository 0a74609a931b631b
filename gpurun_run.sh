mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fullorder_gpu.py -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/variants.log
for v in "warp X=1" "kshare PICROM_WARP_HIST=0"; do
  set -- $v; name=$1; shift
  for c in C5; do
    echo "== $name $c" >> gpurun_out/variants.log
    env "$@" timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-rom --e2e-steps 2 2>&1 | tee -a gpurun_out/variants_raw.log | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step'], d['roofline']['frac'])" >> gpurun_out/variants.log 2>&1
  done
done
echo done
