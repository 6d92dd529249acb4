set -x
OUT=gpurun_out/r02b; mkdir -p $OUT
python tools/cta_timeline.py > $OUT/cta_timeline.txt 2>&1
python tools/acct_conv.py > $OUT/acct_conv.txt 2>&1
bash tools/ncu_profile.sh r02b 4 conv
