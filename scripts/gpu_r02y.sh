set -x
O=gpurun_out/r02y
mkdir -p $O
MLRA_SK=0 MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/trace_mma.py row > $O/trace_mma.txt 2>&1
MLRA_SK=0 MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/timeline.py 11008 4096 3 4096 fwd all > $O/timeline_fwd.txt 2>&1
MLRA_SK=0 MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/timeline.py 11008 4096 3 4096 dx all > $O/timeline_dx.txt 2>&1
