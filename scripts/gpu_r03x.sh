set -x
O=gpurun_out/r03x
mkdir -p $O
MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/timeline.py 11008 4096 3 1024 fwd all > $O/tl_11008_fwd_1k.txt 2>&1
MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/timeline.py 4096 11008 3 1024 dx all > $O/tl_4096_dx_1k.txt 2>&1
