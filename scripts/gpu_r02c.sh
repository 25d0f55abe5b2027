# Verify the split pair-kernel families (whole-tile kernel without stream-K code), A/B vs round 1, small-m timelines.
set -x
O=gpurun_out/r02c
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for i in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline --no-parity --steps 20 > $O/new_$i.json 2> $O/new_$i.err
  (cd scripts/var/r01 && timeout 300 python bench.py --no-cpu-baseline --steps 20) > $O/old_$i.json 2> $O/old_$i.err
done
MS=512,1024 timeout 600 python scripts/sk_probe.py > $O/sk_probe.txt 2>&1
for sk in 2 0 1 4; do
  MLRA_SK=$sk MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/timeline.py 4096 4096 4 512 fwd > $O/timeline_cfg1_sk$sk.txt 2>&1
done
for g in 1 3; do
  MLRA_GEMM=$g MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/trace1.py 4096 4096 4 512 fwd > $O/trace1_cfg1_g$g.txt 2>&1
done
