set -x
O=gpurun_out/r02x
mkdir -p $O
for i in 1 2 3 4; do
  timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/cfg2_$i.json 2> $O/cfg2_$i.err
done
nvidia-smi -q -d CLOCK,PERFORMANCE > $O/smi.txt 2>&1
