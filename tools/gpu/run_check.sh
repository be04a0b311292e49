set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r1s3_pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/r1s3_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r1s3_bench.json 2> gpurun_out/r1s3_bench.err
timeout 300 python tools/ab_phases.py c1_500k 30 > gpurun_out/r1s3_phases.log 2>&1
tail -3 gpurun_out/r1s3_pytest.log; cat gpurun_out/r1s3_bench.json; cat gpurun_out/r1s3_phases.log
