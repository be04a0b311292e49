#!/bin/bash
# A/B of experiment builds (tools/build_variant.py variants/var_NAME ...): the in-tree liblgs.so, then each
# variants/var_*/liblgs.so swapped in, one short bench each.  Usage: [CONFIG=c1] bash tools/gpu/variants.sh
mkdir -p gpurun_out/ab
cp paper_2511_16144_b200/liblgs.so gpurun_out/ab/base.so
CONFIG=${CONFIG:-c1_500k}
if [ -n "$MAPPING" ]; then  # the mapping step's eager (unfused) kernels instead
run() {
  python bench.py --config $CONFIG --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-pruning \
    --multiview none 2>/dev/null | \
    tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read())['mapping_step']; print('$1', d['value'], {k: v['ms'] for k, v in d['phases'].items() if k in ('blend_fwd', 'blend_bwd', 'mapping_loss')})"
}
else
run() {
  python bench.py --config $CONFIG --steps 30 --warmup 5 --no-e2e --no-mapping --no-cpu-baseline --no-pruning \
    --multiview none 2>/dev/null | \
    tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['roofline']['phases']['blend_fused']['ms'], d['clocks'].get('sm_mhz'), d['work']['listed'], {k: v['ms'] for k, v in d['roofline']['phases'].items() if k != 'blend_fused'})"
}
fi
run base
for v in variants/var_*/; do
  cp $v/liblgs.so paper_2511_16144_b200/liblgs.so
  run $(basename $v)
done
cp gpurun_out/ab/base.so paper_2511_16144_b200/liblgs.so
run base_again
