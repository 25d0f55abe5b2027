set -x
O=gpurun_out/r03d
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "arena or graph or capture" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python scripts/sweep.py cfg1 cfg2 cfg3 cfg3_1k cfg4_b3 > $O/sweep_new.jsonl 2>&1
MLRA_GRAPH_SIDE=1 timeout 900 python scripts/sweep.py cfg1 cfg2 cfg3 cfg3_1k cfg4_b3 > $O/sweep_old.jsonl 2>&1
