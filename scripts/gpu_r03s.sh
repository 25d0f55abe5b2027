set -x
O=gpurun_out/r03s
mkdir -p $O
for i in 1 2; do
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_$i.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_$i.log
done
for w in cfg1 cfg2 cfg3 cfg4; do
  timeout 600 python bench.py --workload $w --graph --no-cpu-baseline > $O/graph_$w.json 2> $O/graph_$w.err
done
