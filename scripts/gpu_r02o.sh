set -x
O=gpurun_out/r02o
mkdir -p $O
for i in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/side_$i.json 2> /dev/null
  MLRA_NO_SIDE=1 timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/noside_$i.json 2> /dev/null
done
for i in 1 2; do
  timeout 300 python bench.py --workload cfg1 --graph --no-cpu-baseline --no-parity > $O/cfg1_side_$i.json 2> /dev/null
  MLRA_NO_SIDE=1 timeout 300 python bench.py --workload cfg1 --graph --no-cpu-baseline --no-parity > $O/cfg1_noside_$i.json 2> /dev/null
done
timeout 300 python scripts/sweep.py cfg3_1k > $O/cfg3_1k_side.jsonl 2>&1
MLRA_NO_SIDE=1 timeout 300 python scripts/sweep.py cfg3_1k > $O/cfg3_1k_noside.jsonl 2>&1
