# side-stream schedule A/B after the fused row product
set -x
O=gpurun_out/r04f
mkdir -p $O
for i in 1 2 3; do
  for e in "" MLRA_DA_EARLY=0 MLRA_NO_SIDE=1; do
    tag=${e:-default}; tag=${tag//=/_}
    env $e timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/cfg2_${tag}_$i.json 2> /dev/null
    env $e timeout 300 python scripts/sweep.py cfg3_1k > $O/cfg3_1k_${tag}_$i.jsonl 2>&1
  done
done
MLRA_DA_EARLY=0 timeout 300 python scripts/step_timeline.py cfg2 $O/cfg2_da0_trace.json > $O/cfg2_da0_tl.txt 2>&1
gzip -f $O/*.json
