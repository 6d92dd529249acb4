# final round-2 captures: ncu (cold L2) of the configs[4] step's conv + map kernels, the
# configs[1] convs, launch lists, step timelines
set -x
rm -rf gpurun_out/r02z gpurun_out/r02z_c1; mkdir -p gpurun_out/r02z
timeout 300 python tools/step_timeline.py 1 4 2>&1 | grep -v Warn | tail -19 > gpurun_out/r02z/timeline4.txt
timeout 300 python tools/step_timeline.py 1 1 2>&1 | grep -v Warn | tail -14 > gpurun_out/r02z/timeline1.txt
bash tools/ncu_profile.sh r02z 4 all
bash tools/ncu_profile.sh r02z_c1 1 conv
