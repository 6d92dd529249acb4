OUT=gpurun_out/r02d; mkdir -p $OUT
python tools/acct_conv.py 1 > $OUT/acct_conv1.txt 2>&1
python tools/cta_timeline.py > $OUT/cta_timeline.txt 2>&1
cat $OUT/acct_conv1.txt $OUT/cta_timeline.txt
