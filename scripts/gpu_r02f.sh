set -x
O=gpurun_out/r02f
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_bench_configs.py -m gpu -x -q -p no:cacheprovider -k "stream_k or cfg1 or cfg3 or splitk" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
MS=512,1024 timeout 600 python scripts/sk_probe.py > $O/sk_probe.txt 2>&1
for sk in 4 5; do
  MLRA_SK=$sk MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/timeline.py 4096 4096 4 512 fwd > $O/timeline_cfg1_sk$sk.txt 2>&1
done
timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --graph > $O/cfg1_graph.json 2> $O/cfg1_graph.err
