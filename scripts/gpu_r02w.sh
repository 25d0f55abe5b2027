set -x
O=gpurun_out/r02w
mkdir -p $O
MLRA_HOSTPROF=1 timeout 300 python scripts/host_probe.py > $O/host.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for i in 1 2; do
  timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --no-parity > $O/cfg1_$i.json 2> /dev/null
  timeout 300 python bench.py --workload cfg1 --graph --no-cpu-baseline --no-parity > $O/cfg1g_$i.json 2> /dev/null
  timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/cfg2_$i.json 2> /dev/null
done
timeout 300 python scripts/sweep.py cfg3_1k cfg1 > $O/sweep.jsonl 2>&1
