#!/bin/bash
# Blend-kernel iteration: GPU tests of the blend paths, a short bench, and an ncu capture of the fused
# kernel only (eager fused step, FUSED=1).  Usage: bash tools/gpu/r2_blend.sh <tag>
tag=${1:-blend}
mkdir -p gpurun_out/$tag
python -m pytest tests/test_gpu_plan.py tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -q -x > gpurun_out/$tag/tests.log 2>&1
echo "rc=$?" >> gpurun_out/$tag/tests.log
python bench.py --steps 30 --warmup 5 --no-e2e --no-mapping --no-cpu-baseline --multiview none > gpurun_out/$tag/bench.json 2> gpurun_out/$tag/bench.err
FUSED=1 timeout 300 python tools/profile_step.py c1_500k 1 > gpurun_out/$tag/plain.log 2>&1 && \
FUSED=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:blend_fused -c 1 \
  -o gpurun_out/$tag/fused -f python tools/profile_step.py c1_500k 1 > gpurun_out/$tag/ncu.log 2>&1
tail -2 gpurun_out/$tag/ncu.log
