#!/bin/bash
# Round-end evidence in one GPU call: GPU tests, smoke, cold-L2 ncu captures of the configs[4]
# step (conv + map kernels) and the configs[1] convs, launch lists, step timeline.
# usage: tools/final_capture.sh TAG
TAG=${1:-final}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi > $OUT/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
tail -2 $OUT/smoke.log
bash tools/ncu_profile.sh ${TAG}/ncu_c4 4 all
bash tools/ncu_profile.sh ${TAG}/ncu_c1 1 conv
timeout 300 python tools/step_timeline.py 3 4 > $OUT/step_timeline_c4.txt 2>&1
timeout 300 python tools/step_timeline.py 3 1 > $OUT/step_timeline_c1.txt 2>&1
ls $OUT
