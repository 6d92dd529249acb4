#!/bin/bash
# Quick GPU iteration: conv parity tests + short bench lines (configs[4] and [1]).
# usage: tools/quick.sh TAG [pytest -k expr] [extra env assignments for an A/B line]
TAG=${1:-quick}; KEXPR=${2:-conv or configs}; AB=${3:-}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "$KEXPR" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
for cfg in 4 1; do
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-extras --no-cpu-baseline --no-e2e > $OUT/bench_c$cfg.json 2> $OUT/bench_c$cfg.err
  python -c "import json;d=json.load(open('$OUT/bench_c$cfg.json'));print('cfg$cfg',d['value'],d['ms_per_step'],d['phases_us'])"
  if [ -n "$AB" ]; then
    env $AB timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-extras --no-cpu-baseline --no-e2e > $OUT/bench_c${cfg}_ab.json 2>/dev/null
    python -c "import json;d=json.load(open('$OUT/bench_c${cfg}_ab.json'));print('cfg$cfg AB($AB)',d['value'],d['ms_per_step'],d['phases_us'])"
  fi
done
