# Per-kernel durations of the captured bench step: bash tools/gpu/launches_plan.sh <tag> [ENV=v ...]
tag=${1:-plan_launches}
shift
env "$@" timeout 300 python tools/profile_plan.py c1_500k 3 > gpurun_out/${tag}_plain.log 2>&1 || exit 1
cat gpurun_out/${tag}_plain.log
env "$@" timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --graph-profiling node \
  --log-file gpurun_out/${tag}.csv python tools/profile_plan.py c1_500k 3 > gpurun_out/${tag}.log 2>&1
python tools/launch_table.py gpurun_out/${tag}.csv 4
