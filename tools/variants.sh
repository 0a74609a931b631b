# usage: bash tools/variants.sh NAME... -- compare library variants (built by
# tools/build_variant.py) on the C2 and C5 bench lines; default library first
mkdir -p gpurun_out
out=gpurun_out/variants.log
: > $out
for v in default "$@"; do
  if [ "$v" = default ]; then lib=""; else lib="PICROM_LIB=paper_2201_05555_b200/variants/libpicrom_$v.so"; fi
  for cfg in C2 C5; do
    steps=20; [ $cfg = C5 ] && steps=5
    r=$(env $lib timeout 300 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline --no-rom 2>&1 | tail -1)
    echo "$v $cfg $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,2), "G", round(d["roofline"]["frac"],4), "e2e", round(d["e2e"]["value"]/1e9,2))' 2>&1)" >> $out
  done
done
cat $out
