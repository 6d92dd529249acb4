#!/bin/bash
# ncu --set full captures of the hot kernels of one bench step (warm caches as in the run),
# plus the launch list of the same bench command.  Output: gpurun_out/$TAG/.
# usage: tools/ncu_profile.sh TAG
TAG=${1:-prof}
OUT=gpurun_out/$TAG
mkdir -p $OUT
cap() {  # name regex skip
  timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:$2 -s $3 -c 1 \
    -o $OUT/$1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/$1.log 2>&1
  echo "$1: $(tail -1 $OUT/$1.log)"
}
cap conv_fwd k_conv_umma 2
cap conv_dgrad k_conv_umma 3
cap conv_wgrad k_wgrad_umma 1
cap kmap_probe k_probe 2
cap kmap_emit k_emit 2
cap quant_insert k_insert 2
cap quant_rank k_rank 2
cap kmap_sort k_radix_sort_coop 2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls $OUT
