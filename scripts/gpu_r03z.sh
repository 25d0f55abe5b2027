# graph-vs-eager probe (cfg3 shapes at 8192 tokens) + lazy owner-count rebuild A/B
set -x
O=gpurun_out/r03z
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "stream_k" > $O/parity.log 2>&1; echo "rc=$?" >> $O/parity.log
for e in "" MLRA_PDL=0 MLRA_DA_EARLY=0 MLRA_NO_SIDE=1; do
  env $e timeout 300 python scripts/graph_probe.py 11008 4096 8192 >> $O/graph_probe.jsonl 2>> $O/graph_probe.err
done
timeout 300 python scripts/graph_probe.py 4096 11008 8192 >> $O/graph_probe.jsonl 2>> $O/graph_probe.err
timeout 300 python scripts/graph_probe.py 4096 4096 8192 >> $O/graph_probe.jsonl 2>> $O/graph_probe.err
timeout 300 python scripts/graph_probe.py 11008 4096 4096 >> $O/graph_probe.jsonl 2>> $O/graph_probe.err
for v in 0 1; do
  MLRA_SK_OWNER4=$v MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/timeline.py 11008 4096 3 1024 fwd all > $O/tl_fwd_o4$v.txt 2>&1
done
for i in 1 2; do
  for v in 0 1; do
    MLRA_SK_OWNER4=$v timeout 300 python scripts/sweep.py cfg3_1k > $O/cfg3_1k_o4${v}_$i.jsonl 2>&1
  done
done
cat $O/graph_probe.jsonl; tail -3 $O/graph_probe.err
