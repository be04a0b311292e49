# Round-end evidence: bench line, ncu --set full of one fused eager step, launch list.
#   bash tools/gpu/final_profile.sh <tag>
tag=${1:-final}
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
head -c 400 gpurun_out/${tag}_bench.json; echo
FUSED=1 bash tools/gpu/ncu_step.sh ${tag}_ncu
FUSED=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launches.csv python tools/profile_step.py c1_500k 3 > gpurun_out/${tag}_launches.log 2>&1
python tools/launch_table.py gpurun_out/${tag}_launches.csv 3
