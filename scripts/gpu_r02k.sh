set -x
O=gpurun_out/r02k
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for s in "11008 4096 4096 16" "4096 11008 4096 16" "4096 4096 512 8" "4096 4096 1024 8"; do
  MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/thin_timeline.py $s > "$O/thin_$(echo $s | tr ' ' _).txt" 2>&1
done
timeout 300 python scripts/skinny_probe.py > $O/skinny.txt 2>&1
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/cfg2_$i.json 2> /dev/null
timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --no-parity --graph > $O/cfg1g_$i.json 2> /dev/null
done
timeout 600 python scripts/sweep.py cfg3_1k cfg3 > $O/sweep.jsonl 2>&1
