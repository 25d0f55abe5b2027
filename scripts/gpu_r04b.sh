# cluster row-product kernel: parity, step timelines, A/B against the range kernel
set -x
O=gpurun_out/r04b
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "cluster or launch_switches or bitwise" > $O/parity.log 2>&1; echo "rc=$?" >> $O/parity.log
timeout 300 python scripts/step_timeline.py cfg2 $O/cfg2_trace.json > $O/cfg2_tl.txt 2>&1
MLRA_THIN_CL=0 timeout 300 python scripts/step_timeline.py cfg2 $O/cfg2_cl0_trace.json > $O/cfg2_cl0_tl.txt 2>&1
gzip -f $O/*.json
for i in 1 2; do
  for v in 1 0; do
    MLRA_THIN_CL=$v timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/cfg2_cl${v}_$i.json 2> /dev/null
    MLRA_THIN_CL=$v timeout 300 python scripts/sweep.py cfg3_1k cfg4_b3 > $O/sweep_cl${v}_$i.jsonl 2>&1
  done
done
tail -n 3 $O/parity.log
