set -x
O=gpurun_out/r02z
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_bench_configs.py -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
MLRA_SK=0 MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/trace_mma.py row > $O/trace_mma_tr.txt 2>&1
MLRA_EPI_TR=0 MLRA_SK=0 MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/trace_mma.py row > $O/trace_mma_old.txt 2>&1
for i in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/tr_$i.json 2> /dev/null
  MLRA_EPI_TR=0 timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/old_$i.json 2> /dev/null
done
MS=4096,1024 timeout 900 python scripts/sk_probe.py > $O/sk_probe.txt 2>&1
