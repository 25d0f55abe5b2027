set -x
O=gpurun_out/r02r
mkdir -p $O
MS=4096,2048 timeout 900 python scripts/sk_probe.py > $O/sk_probe.txt 2>&1
