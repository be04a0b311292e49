# One headline step under ncu --set full with source correlation (tools/profile_step.py), for the
# summaries under profiles/.  Usage: bash tools/gpu/ncu_step.sh <tag>
tag=${1:-step}
timeout 300 python tools/profile_step.py c1_500k 1 > gpurun_out/${tag}_plain.log 2>&1 || exit 1
timeout 1500 ncu --set full --import-source on --clock-control none -o gpurun_out/${tag} -f \
  python tools/profile_step.py c1_500k 1 > gpurun_out/${tag}_ncu.log 2>&1
tail -3 gpurun_out/${tag}_ncu.log
