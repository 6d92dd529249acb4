#!/bin/bash
# A/B of environment knobs on short bench lines.
# usage: tools/ab_env.sh TAG "CFGS" "ENV1" "ENV2" ...   (ENV = space-separated assignments or "-" for default)
TAG=$1; CFGS=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
i=0
for AB in "$@"; do
  for cfg in $CFGS; do
    E=""; [ "$AB" != "-" ] && E="$AB"
    env $E timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-extras --no-cpu-baseline --no-e2e > $OUT/b_${i}_c$cfg.json 2> $OUT/b_${i}_c$cfg.err
    python -c "import json;d=json.load(open('$OUT/b_${i}_c$cfg.json'));print('cfg$cfg [$AB]',round(d['value'],1),round(d['ms_per_step'],4),{k:round(v) for k,v in d['phases_us'].items()})" || tail -3 $OUT/b_${i}_c$cfg.err
  done
  i=$((i+1))
done
