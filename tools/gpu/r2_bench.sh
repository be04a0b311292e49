#!/bin/bash
# Round-2 GPU session: full GPU tests, the default bench line, per-config lines (c0, c1, c2, c4), the
# reference arm, and one ncu launch list per config (cold-cache, serialised: kernel SHARES of the step,
# not absolute times); outputs under gpurun_out/r2/.
set -x
mkdir -p gpurun_out/r2
python -m pytest tests -m gpu -q > gpurun_out/r2/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/gpu_tests.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2/bench_default.json 2> gpurun_out/r2/bench_default.err
for c in c0 c1 c2 c4; do
  python bench.py --config $c --steps 20 --warmup 5 --no-mapping --no-pruning > gpurun_out/r2/bench_$c.json 2> gpurun_out/r2/bench_$c.err
done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2/bench_ref.json 2> gpurun_out/r2/bench_ref.err
for c in c1_500k c0 c1 c2 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r2/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-e2e \
    --no-mapping --no-cpu-baseline --no-pruning --multiview none > gpurun_out/r2/launches_$c.log 2>&1
done
