set -x
O=gpurun_out/r02j
mkdir -p $O
for s in "11008 4096 4096 16" "4096 11008 4096 16" "4096 4096 512 8" "4096 4096 1024 8"; do
  MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/thin_timeline.py $s > "$O/thin_$(echo $s | tr ' ' _).txt" 2>&1
done
