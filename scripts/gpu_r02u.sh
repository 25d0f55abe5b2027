set -x
O=gpurun_out/r02u
mkdir -p $O
MLRA_HOSTPROF=1 timeout 300 python scripts/host_probe.py > $O/host.txt 2>&1
