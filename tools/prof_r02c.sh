OUT=gpurun_out/r02c; mkdir -p $OUT
python tools/acct_wgrad.py 1 > $OUT/acct_wgrad1.txt 2>&1
python tools/acct_wgrad.py 4 > $OUT/acct_wgrad4.txt 2>&1
python tools/acct_conv.py > $OUT/acct_conv.txt 2>&1
B="python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-extras --no-e2e"
timeout 900 ncu --set full --clock-control none --cache-control all --import-source on -k regex:k_wgrad_umma -s 1 -c 1 -o $OUT/conv_wgrad $B > $OUT/wg.log 2>&1
cat $OUT/acct_wgrad1.txt $OUT/acct_wgrad4.txt
