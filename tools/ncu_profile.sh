#!/bin/bash
# ncu --set full captures of the hot kernels of one bench step, plus the launch list of the
# same bench command.  --cache-control all: L2 is flushed before each replayed pass, so DRAM
# bytes are those of a cold-L2 launch (the bench flushes L2 before every step).
# usage: tools/ncu_profile.sh TAG CONFIG [kernel-set]
TAG=${1:-prof}; CFG=${2:-4}; SET=${3:-all}
OUT=gpurun_out/$TAG
mkdir -p $OUT
B="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-extras --no-e2e"
cap() {  # name regex skip
  timeout 900 ncu --set full --clock-control none --cache-control all --import-source on -k regex:$2 -s $3 -c 1 \
    -o $OUT/$1 $B > $OUT/$1.log 2>&1
  echo "$1: $(tail -1 $OUT/$1.log | head -c 200)"
}
# launch order per step: fwd conv (k_conv_umma), dgrad conv (k_conv_umma), wgrad; the
# Workload setup runs one untimed map build; warm-up 1 step
if [ "$SET" = all ] || [ "$SET" = conv ]; then
cap conv_fwd k_conv_umma 2
cap conv_dgrad k_conv_umma 3
cap conv_wgrad k_wgrad_umma 1
fi
# map-build kernels: configs[4]'s setup builds 16 per-scan maps (LPT costs) before the
# full-size builds, so skip those
MS=1; [ "$CFG" = 4 ] && MS=16
if [ "$SET" = all ] || [ "$SET" = map ]; then
cap kmap_probe k_probe $MS
cap kmap_emit k_emit $MS
cap quant_insert k_insert $MS
cap quant_rank k_rank $MS
cap kmap_sort k_radix_sort_coop $MS
fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $OUT/launches.csv $B > /dev/null 2>&1
ls $OUT
