#!/bin/bash
# A/B of speculative plans (capture without the layered second pass) on every config: on / off / on
run() {
  python bench.py --config $1 --steps 30 --warmup 5 --no-e2e --no-mapping --no-cpu-baseline --no-pruning \
    --multiview none $2 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', '${2:-speculative}', d['value'], d['ms_per_step'], d['plan'], d['gpu_launches'], d['clocks'].get('sm_mhz'))"
}
for c in ${CONFIGS:-c1_500k c0 c1 c2 c4}; do
  run $c
  run $c --no-speculative-plans
  run $c
done
