set -x
O=gpurun_out/r02s
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_bench_configs.py -m gpu -x -q -p no:cacheprovider -k "hybrid or stream_k or cfg2 or cfg1" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
MS=4096,2048 timeout 900 python scripts/sk_probe.py > $O/sk_probe.txt 2>&1
for i in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/hyb_$i.json 2> /dev/null
  MLRA_SK=0 timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/whole_$i.json 2> /dev/null
done
