set -x
O=gpurun_out/r02e
mkdir -p $O
for m in 512 1024; do
  MLRA_SK=4 MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/timeline.py 4096 4096 4 $m fwd > $O/timeline_split_4096_m$m.txt 2>&1
done
MLRA_SK=4 MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/timeline.py 11008 4096 3 512 fwd > $O/timeline_split_11008_m512.txt 2>&1
