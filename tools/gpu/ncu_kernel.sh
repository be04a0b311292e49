# ncu --set full of one kernel of one eager headline step: bash tools/gpu/ncu_kernel.sh <tag> <kernel regex>
tag=$1; k=$2
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o gpurun_out/$tag -f \
  python tools/profile_step.py c1_500k 1 > gpurun_out/${tag}_ncu.log 2>&1
tail -2 gpurun_out/${tag}_ncu.log
