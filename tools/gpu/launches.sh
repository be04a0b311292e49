# Per-kernel durations of one headline step (ncu launch list, no replay sets):
#   bash tools/gpu/launches.sh <tag> [extra env]
tag=${1:-launches}
shift
env "$@" timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}.csv python tools/profile_step.py c1_500k 3 > gpurun_out/${tag}.log 2>&1
python tools/launch_table.py gpurun_out/${tag}.csv 3
