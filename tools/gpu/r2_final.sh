#!/bin/bash
# End-of-round GPU session: GPU tests, smoke, the default bench line, per-config lines (c0, c1, c2, c4),
# the reference arm, and the launch list of each config's timed plan replays (ncu, cold-cache and
# serialised: kernel SHARES of the step, not absolute times).  Outputs under gpurun_out/fin/.
set -x
mkdir -p gpurun_out/fin
if [ -z "$SKIP_TESTS" ]; then
  python -m pytest tests -m gpu -q > gpurun_out/fin/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fin/gpu_tests.log
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/fin/smoke.log
fi
python bench.py > gpurun_out/fin/bench_default.json 2> gpurun_out/fin/bench_default.err
for c in c0 c1 c2 c4; do
  python bench.py --config $c --steps 20 --warmup 5 --no-mapping --no-pruning > gpurun_out/fin/bench_$c.json 2> gpurun_out/fin/bench_$c.err
done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin/bench_ref.json 2> gpurun_out/fin/bench_ref.err
for c in c1_500k c0 c1 c2 c4; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/fin/launches_$c.csv python bench.py --config $c --steps 3 --warmup 3 --no-e2e \
    --no-mapping --no-cpu-baseline --no-pruning --multiview none > gpurun_out/fin/launches_$c.log 2>&1
done
