set -x
O=gpurun_out/r03i
mkdir -p $O
MLRA_DA_EARLY=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_bench_configs.py -m gpu -q -x -p no:cacheprovider -k "cfg2 or cfg1 or bitwise or arena" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for i in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/base_$i.json 2> /dev/null
  MLRA_DA_EARLY=1 timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/early_$i.json 2> /dev/null
done
for i in 1 2; do
  timeout 300 python bench.py --workload cfg1 --graph --no-cpu-baseline --no-parity > $O/cfg1_base_$i.json 2> /dev/null
  MLRA_DA_EARLY=1 timeout 300 python bench.py --workload cfg1 --graph --no-cpu-baseline --no-parity > $O/cfg1_early_$i.json 2> /dev/null
done
timeout 600 python scripts/sweep.py cfg3 cfg3_1k cfg4_b3 > $O/sweep_base.jsonl 2>&1
MLRA_DA_EARLY=1 timeout 600 python scripts/sweep.py cfg3 cfg3_1k cfg4_b3 > $O/sweep_early.jsonl 2>&1
