# streamed row product (tile flags from the producing GEMM): parity first, short timeouts
set -x
O=gpurun_out/r04g
mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "chained or cluster" > $O/t1.log 2>&1; echo "rc=$?" >> $O/t1.log
tail -n 3 $O/t1.log
grep -q "rc=0" $O/t1.log || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_bench_configs.py -m gpu -x -q -p no:cacheprovider > $O/parity.log 2>&1; echo "rc=$?" >> $O/parity.log
timeout 300 python scripts/step_timeline.py cfg2 $O/cfg2_trace.json > $O/cfg2_tl.txt 2>&1
gzip -f $O/*.json
for i in 1 2 3; do
  for v in 1 0; do
    MLRA_STREAM_ROWS=$v timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/cfg2_s${v}_$i.json 2> /dev/null
  done
done
tail -n 3 $O/parity.log
