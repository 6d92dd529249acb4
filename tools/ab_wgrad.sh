for cfg in 1 4; do
for v in "" "MK_WGRAD_GA=2" "MK_WGRAD_GA=4" "MK_WGRAD_NP=8" "MK_WGRAD_NP=8 MK_WGRAD_GA=2"; do
  env $v timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('cfg$cfg', '$v', d['phases_us']['conv_wgrad'])"
done; done
