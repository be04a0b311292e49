#!/bin/bash
# Launch lists of the captured plan's replays (speculative plans have no conditional node, so ncu
# lists their kernel nodes): bench.py's timed step under ncu, cold-cache and serialised.
mkdir -p gpurun_out/r2p
for c in ${CONFIGS:-c1_500k c2 c4}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/r2p/launches_$c.csv python bench.py --config $c --steps 3 --warmup 3 --no-e2e \
    --no-mapping --no-cpu-baseline --no-pruning --multiview none > gpurun_out/r2p/launches_$c.log 2>&1
done
