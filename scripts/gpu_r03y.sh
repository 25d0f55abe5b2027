# stream-K owner fix-up on all 16 warps: parity, timelines, A/B (MLRA_SK_OWNER4=1 = old path)
set -x
O=gpurun_out/r03y
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "stream_k" > $O/parity.log 2>&1; echo "rc=$?" >> $O/parity.log
timeout 900 python -m pytest tests/test_bench_configs.py -m gpu -x -q -p no:cacheprovider -k "streamk or default" > $O/cfgs.log 2>&1; echo "rc=$?" >> $O/cfgs.log
for v in 0 1; do
  MLRA_SK_OWNER4=$v MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/timeline.py 11008 4096 3 1024 fwd all > $O/tl_fwd_o4$v.txt 2>&1
  MLRA_SK_OWNER4=$v MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/timeline.py 4096 11008 3 1024 dx all > $O/tl_dx_o4$v.txt 2>&1
done
for i in 1 2 3; do
  for v in 0 1; do
    MLRA_SK_OWNER4=$v timeout 300 python scripts/sweep.py cfg3_1k > $O/cfg3_1k_o4${v}_$i.jsonl 2>&1
  done
done
for v in 0 1; do
  MLRA_SK_OWNER4=$v timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/cfg2_o4$v.json 2> /dev/null
done
tail -n 3 $O/*.log
