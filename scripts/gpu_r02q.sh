set -x
O=gpurun_out/r02q
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_bench_configs.py tests/test_train.py -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for i in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/new_$i.json 2> /dev/null
  MLRA_SIDE_FIRST=1 timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/old_$i.json 2> /dev/null
done
for i in 1 2; do
  timeout 300 python bench.py --workload cfg1 --graph --no-cpu-baseline --no-parity > $O/cfg1_new_$i.json 2> /dev/null
  MLRA_SIDE_FIRST=1 timeout 300 python bench.py --workload cfg1 --graph --no-cpu-baseline --no-parity > $O/cfg1_old_$i.json 2> /dev/null
  timeout 300 python bench.py --workload cfg4 --no-cpu-baseline --no-parity > $O/cfg4_new_$i.json 2> /dev/null
  MLRA_SIDE_FIRST=1 timeout 300 python bench.py --workload cfg4 --no-cpu-baseline --no-parity > $O/cfg4_old_$i.json 2> /dev/null
done
timeout 300 python scripts/sweep.py cfg3_1k cfg3 > $O/cfg3_new.jsonl 2>&1
MLRA_SIDE_FIRST=1 timeout 300 python scripts/sweep.py cfg3_1k cfg3 > $O/cfg3_old.jsonl 2>&1
