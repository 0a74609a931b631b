mkdir -p gpurun_out
: > gpurun_out/variants.log
for rep in 1 2; do
for v in main dsetp; do
  if [ "$v" = main ]; then L="X=1"; else L="PICROM_LIB=paper_2201_05555_b200/variants/libpicrom_$v.so"; fi
  for c in C2 C5; do
    echo "== $v $c" >> gpurun_out/variants.log
    env $L timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step'], d['roofline']['frac'])" >> gpurun_out/variants.log 2>&1
  done
done
done
./tools/bin/fp64_peak > gpurun_out/fp64_peak.log 2>&1
python - > gpurun_out/dgemm.log 2>&1 <<'PY'
import torch, time
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(f"dgemm {n}: {best:.3f} ms  {2*n**3/best/1e9:.1f} TF/s")
PY
echo done
