#!/bin/bash
# Launch lists (ncu, cold-cache, serialised) of the timed plan replays: the in-tree liblgs.so and
# each variants/var_*/liblgs.so.  Usage: [CONFIG=c1_500k] bash tools/gpu/ab_launches.sh
mkdir -p gpurun_out/abl
CONFIG=${CONFIG:-c1_500k}
cp paper_2511_16144_b200/liblgs.so gpurun_out/abl/base.so
one() {
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/abl/$1_$CONFIG.csv python bench.py --config $CONFIG --steps 3 --warmup 3 --no-e2e \
    --no-mapping --no-cpu-baseline --no-pruning --multiview none > gpurun_out/abl/$1_$CONFIG.log 2>&1
}
one base
for v in variants/var_*/; do
  cp $v/liblgs.so paper_2511_16144_b200/liblgs.so
  one $(basename $v)
done
cp gpurun_out/abl/base.so paper_2511_16144_b200/liblgs.so
