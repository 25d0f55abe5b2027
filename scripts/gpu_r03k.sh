set -x
O=gpurun_out/r03k
mkdir -p $O
MLRA_SK=6 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "llama or stream_k or bitwise" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for i in 1 2; do
  MLRA_SK=6 timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/alt_$i.json 2> /dev/null
  timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/cur_$i.json 2> /dev/null
  MLRA_LIB=scripts/var/prev/libmlra.so timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/prev_$i.json 2> /dev/null
done
MS=4096 timeout 600 python scripts/sk_probe.py > $O/sk_cur.txt 2>&1
