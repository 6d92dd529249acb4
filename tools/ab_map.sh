# A/B of map-build compile-time variants (build_variants/libmk_<v>.so) on configs[4] and [1]
for cfg in 4 1; do
for v in ${VARIANTS:-"" r8 r12 r16 p4 p1}; do
  L=""; [ -n "$v" ] && L="MK_LIBRARY=build_variants/libmk_$v.so"
  env $L timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); ph=d['phases_us']; print('cfg$cfg', '${v:-base}', ph.get('quantize'), ph.get('kmap'), round(ph.get('quantize')+ph.get('kmap'),1))"
done; done
