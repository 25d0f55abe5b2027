set -x
O=gpurun_out/r02t
mkdir -p $O
timeout 300 python scripts/host_probe.py > $O/host.txt 2>&1
timeout 300 python scripts/h2d_probe.py > $O/h2d.txt 2>&1
