#!/bin/bash
# GPU tests, then variants.sh (in-tree lib vs variants/var_*) on the layered configs
mkdir -p gpurun_out/abl
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in ${CONFIGS:-c1_500k c2 c4 c1}; do CONFIG=$c bash tools/gpu/variants.sh; done
