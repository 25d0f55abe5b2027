# fused row product gated on tokens (> 512): cfg1 default (range kernel now) vs
# MLRA_THIN_CL=1 (fused forced); cluster / launch-switch tests
set -x
O=gpurun_out/r05d
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "cluster or launch_switches or bitwise" > $O/t.log 2>&1; echo "rc=$?" >> $O/t.log
for i in 1 2 3; do
  timeout 300 python scripts/sweep.py cfg1 cfg3_1k > $O/sweep_default_$i.jsonl 2>&1
  MLRA_THIN_CL=1 timeout 300 python scripts/sweep.py cfg1 cfg3_1k > $O/sweep_cl1_$i.jsonl 2>&1
done
timeout 300 python scripts/step_timeline.py cfg1 $O/cfg1_trace.json > $O/cfg1_tl.txt 2>&1
tail -n 2 $O/t.log
