#!/bin/bash
# compute-sanitizer over the fused step: memcheck / racecheck / synccheck on the eager fused step
# (FUSED=1) and memcheck on the captured plan, config c0 (small).  Output: gpurun_out/sanitize/.
mkdir -p gpurun_out/sanitize
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  FUSED=1 timeout 1200 $S --tool $tool --error-exitcode 9 python tools/profile_step.py c0 1 \
    > gpurun_out/sanitize/eager_$tool.log 2>&1
  echo "eager $tool rc=$?" >> gpurun_out/sanitize/summary.txt
done
timeout 1200 $S --tool memcheck --error-exitcode 9 python tools/plan_step.py c0 > gpurun_out/sanitize/plan_memcheck.log 2>&1
echo "plan memcheck rc=$?" >> gpurun_out/sanitize/summary.txt
timeout 1200 $S --tool racecheck --error-exitcode 9 python tools/plan_step.py c0 > gpurun_out/sanitize/plan_racecheck.log 2>&1
echo "plan racecheck rc=$?" >> gpurun_out/sanitize/summary.txt
