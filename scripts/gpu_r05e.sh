# per-CTA phases of the fused row product (k_rowmma_cl) at cfg3's 1024-token share and cfg2
set -x
O=gpurun_out/r05e
mkdir -p $O
for s in "4096 4096 1024 8" "11008 4096 1024 8" "4096 11008 1024 8" "11008 4096 4096 16" "4096 4096 4096 16"; do
  MLRA_LIB=scripts/var/libmlra_dev.so timeout 120 python scripts/thin_timeline.py $s > "$O/tl_${s// /_}.txt" 2>&1
done
