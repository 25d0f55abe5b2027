# fused row product: 8-CTA clusters above ~2.4K tokens (shipped) vs 16-CTA clusters always
set -x
O=gpurun_out/r05j
mkdir -p $O
MLRA_LIB=scripts/var/libmlra_c16.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "cluster or chained or bitwise" > $O/t_c16.log 2>&1; echo "rc=$?" >> $O/t_c16.log
for i in 1 2 3; do
  timeout 300 python scripts/sweep.py cfg2 cfg3 > $O/sweep_c8_$i.jsonl 2>&1
  MLRA_LIB=scripts/var/libmlra_c16.so timeout 300 python scripts/sweep.py cfg2 cfg3 > $O/sweep_c16_$i.jsonl 2>&1
done
