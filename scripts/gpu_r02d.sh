# Split-K fix-up by all warps: parity + timing; skinny-product and K1/write-bandwidth probes.
set -x
O=gpurun_out/r02d
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_bench_configs.py -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
MS=512,1024 timeout 600 python scripts/sk_probe.py > $O/sk_probe.txt 2>&1
for sk in 2; do
  MLRA_SK=$sk MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/timeline.py 4096 4096 4 512 fwd > $O/timeline_cfg1_sk$sk.txt 2>&1
done
timeout 300 python scripts/skinny_probe.py > $O/skinny_probe.txt 2>&1
timeout 300 python scripts/write_bw_probe.py > $O/write_bw.txt 2>&1
timeout 300 python scripts/k1_probe.py > $O/k1_probe.txt 2>&1
timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --graph > $O/cfg1_graph.json 2> $O/cfg1_graph.err
timeout 300 python bench.py --no-cpu-baseline > $O/cfg2.json 2> $O/cfg2.err
