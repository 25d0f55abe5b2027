set -x
O=gpurun_out/r03m
mkdir -p $O
timeout 900 python -m pytest tests/test_e8p.py tests/test_cb2.py -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python scripts/sweep.py e8p > $O/sweep.jsonl 2>&1
