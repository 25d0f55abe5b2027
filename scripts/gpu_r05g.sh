# two-deep factor prefetch in the fused row product (fa / fb register ping-pong):
# gpu tests, per-CTA timelines, A/B against the previous build (scripts/var/libmlra_base.so)
set -x
O=gpurun_out/r05g
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/t.log 2>&1; echo "rc=$?" >> $O/t.log
tail -n 2 $O/t.log
for s in "4096 4096 1024 8" "11008 4096 1024 8" "4096 11008 1024 8" "11008 4096 4096 16" "4096 4096 4096 16"; do
  MLRA_LIB=scripts/var/libmlra_dev.so timeout 120 python scripts/thin_timeline.py $s > "$O/tl_${s// /_}.txt" 2>&1
done
for i in 1 2 3; do
  timeout 300 python scripts/sweep.py cfg1 cfg2 cfg3_1k cfg3 cfg4_b3 > $O/sweep_new_$i.jsonl 2>&1
  MLRA_LIB=scripts/var/libmlra_base.so timeout 300 python scripts/sweep.py cfg1 cfg2 cfg3_1k cfg3 cfg4_b3 > $O/sweep_base_$i.jsonl 2>&1
done
