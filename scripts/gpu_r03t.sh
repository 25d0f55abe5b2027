set -x
O=gpurun_out/r03t
mkdir -p $O
timeout 900 python -m pytest tests/test_e8p.py -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python scripts/rht_probe.py > $O/rht_tf32.txt 2>&1
timeout 600 python scripts/sweep.py e8p > $O/sweep.jsonl 2>&1
