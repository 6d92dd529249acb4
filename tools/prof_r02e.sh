OUT=gpurun_out/r02e; mkdir -p $OUT
B="python bench.py --config 1 --steps 1 --warmup 1 --no-cpu-baseline --no-extras --no-e2e"
timeout 900 ncu --set full --clock-control none --cache-control all --import-source on -k regex:k_conv_umma -s 2 -c 1 -o $OUT/conv_fwd $B > $OUT/fwd.log 2>&1
tail -2 $OUT/fwd.log
