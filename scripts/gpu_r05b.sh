# Schedules at 4096 tokens per layer shape (whole tiles vs stream-K vs split-K):
# is the 2-wave whole-tile plan of the 4096x11008 layers (128 tiles over 74 pairs)
# still the cheapest after the all-warp owner fix-up?
set -x
O=gpurun_out/r05b
mkdir -p $O
MS=4096 timeout 600 python scripts/sk_probe.py > $O/sk_4096.jsonl 2> $O/sk_4096.err
MS=2048 timeout 600 python scripts/sk_probe.py > $O/sk_2048.jsonl 2> $O/sk_2048.err
