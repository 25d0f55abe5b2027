set -x
O=gpurun_out/r03a
mkdir -p $O
for c in 8 16 32 1000; do
  for s in "11008 4096 4096 16" "4096 11008 4096 16" "4096 4096 512 8"; do
    MLRA_THIN_MAXC=$c MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/thin_timeline.py $s > "$O/thin_c${c}_$(echo $s | tr ' ' _).txt" 2>&1
  done
  MLRA_THIN_MAXC=$c timeout 300 python scripts/skinny_probe.py > $O/skinny_c$c.txt 2>&1
done
