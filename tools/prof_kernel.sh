#!/bin/bash
# ncu --set full capture of one kernel (regex) in the bench step (warm caches as in the run).
# usage: tools/prof_kernel.sh TAG REGEX [launch-skip]
TAG=$1; K=$2; SKIP=${3:-2}
mkdir -p gpurun_out/$TAG
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:$K -s $SKIP -c 1 \
  -o gpurun_out/$TAG/prof_$K python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/$TAG/ncu_$K.log 2>&1
tail -3 gpurun_out/$TAG/ncu_$K.log
