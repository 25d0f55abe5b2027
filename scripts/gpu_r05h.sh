# early dA only while dY <= 48 MB (default now) vs always early (MLRA_DA_EARLY=1, the previous default)
set -x
O=gpurun_out/r05h
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "launch_switches or chained or bitwise" > $O/t.log 2>&1; echo "rc=$?" >> $O/t.log
tail -n 2 $O/t.log
for i in 1 2 3; do
  timeout 300 python scripts/sweep.py cfg2 cfg3_1k cfg3 cfg4_b3 > $O/sweep_new_$i.jsonl 2>&1
  MLRA_DA_EARLY=1 timeout 300 python scripts/sweep.py cfg2 cfg3_1k cfg3 cfg4_b3 > $O/sweep_early_$i.jsonl 2>&1
done
timeout 300 python scripts/step_timeline.py cfg2 $O/cfg2_trace.json > $O/cfg2_tl.txt 2>&1
gzip -f $O/*.json
