set -x
python -m pytest tests/test_gpu_plan.py -x -q 2>&1 | tail -5
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash tools/gpu/variants.sh
CONFIG=c1 bash tools/gpu/variants.sh
CONFIG=c2 bash tools/gpu/variants.sh
CONFIG=c4 bash tools/gpu/variants.sh
CONFIG=c0 bash tools/gpu/variants.sh
