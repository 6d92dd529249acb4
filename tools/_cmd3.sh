OUT=gpurun_out/r02s3_t3; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --durations=10 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
bash tools/ab_env.sh r02s3_ab2 "4 1 2 3" "-" "MK_FWD_NPW=4" "MK_WGRAD_NP=8" "MK_WGRAD_NP=16"
