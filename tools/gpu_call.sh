#!/bin/bash
# Development GPU call: build, GPU tests (optional -k expression), accounting traces, A/B lines.
# usage: tools/gpu_call.sh TAG [pytest -k expr | all | none] [acct cfg list] [A/B cfgs] [A/B env ...]
TAG=$1; K=${2:-all}; ACCT=${3:-}; CFGS=${4:-"4 1"}; shift 4 2>/dev/null
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
if [ "$K" != "none" ]; then
  if [ "$K" = "all" ]; then KX=(); else KX=(-k "$K"); fi
  timeout 900 python -m pytest tests -m gpu -x -q "${KX[@]}" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  tail -2 $OUT/pytest_gpu.log
fi
for c in $ACCT; do
  timeout 300 python tools/acct_conv.py $c > $OUT/acct_conv_c$c.txt 2>&1; cat $OUT/acct_conv_c$c.txt | tail -16
  timeout 300 python tools/acct_wgrad.py $c > $OUT/acct_wgrad_c$c.txt 2>&1; cat $OUT/acct_wgrad_c$c.txt | tail -22
done
[ $# -gt 0 ] && bash tools/ab_env.sh $TAG/ab "$CFGS" "$@"
exit 0
