set -x
O=gpurun_out/r04i
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "cluster" > $O/t.log 2>&1; echo "rc=$?" >> $O/t.log
timeout 300 python bench.py --workload cfg4 --no-cpu-baseline --no-parity > $O/cfg4.json 2>/dev/null
timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/cfg2.json 2>/dev/null
tail -n 2 $O/t.log
