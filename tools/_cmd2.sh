OUT=gpurun_out/r02s3_fix; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --durations=10 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
MK_FWD_NPW=8 MK_FWD_SAMAX=8 timeout 600 python -m pytest tests -m gpu -x -q -k "conv or configs" > $OUT/pytest_npw8.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_npw8.log
tail -2 $OUT/pytest_npw8.log
bash tools/ab_env.sh r02s3_ab1 "4 1" "-" "MK_FWD_SAMAX=8" "MK_FWD_NPW=8 MK_FWD_SAMAX=8" "MK_FWD_NPW=8" "MK_WGRAD_APAD=1"
