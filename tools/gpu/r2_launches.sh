#!/bin/bash
# Launch lists (ncu gpu__time_duration, cold-cache, serialised) of the fused step per config: the
# captured plan's kernels run uncaptured (FUSED=1 -> LGS_OPT_FUSED_EAGER; ncu cannot list kernel
# nodes of a graph with conditional nodes).  3 steps per config; outputs in gpurun_out/r2l/.
mkdir -p gpurun_out/r2l
for c in c1_500k c0 c1 c2 c4; do
  FUSED=1 timeout 600 python tools/profile_step.py $c 3 > gpurun_out/r2l/plain_$c.log 2>&1 && \
  FUSED=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r2l/launches_$c.csv python tools/profile_step.py $c 3 > gpurun_out/r2l/ncu_$c.log 2>&1
done
