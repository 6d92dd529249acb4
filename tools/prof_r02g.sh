# round-2 profile capture: timeline + bench line + ncu (cold L2) of the configs[4] step and
# the configs[1] conv kernels
set -x
mkdir -p gpurun_out/r02g
timeout 300 python tools/step_timeline.py 1 4 2>&1 | grep -v Warn | tail -19 > gpurun_out/r02g/timeline4.txt
timeout 300 python tools/step_timeline.py 1 1 2>&1 | grep -v Warn | tail -14 > gpurun_out/r02g/timeline1.txt
bash tools/ncu_profile.sh r02g 4 all
bash tools/ncu_profile.sh r02g_c1 1 conv
