# fused row product (in-kernel factor split + post jobs, no prep launch in front)
set -x
O=gpurun_out/r04d
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > $O/parity.log 2>&1; echo "rc=$?" >> $O/parity.log
timeout 300 python scripts/step_timeline.py cfg2 $O/cfg2_trace.json > $O/cfg2_tl.txt 2>&1
timeout 300 python scripts/step_timeline.py cfg3 $O/cfg3_1k_trace.json 1024 > $O/cfg3_1k_tl.txt 2>&1
gzip -f $O/*.json
timeout 300 python scripts/rowmma_probe.py > $O/probe.jsonl 2>/dev/null
for i in 1 2; do
  for v in 1 0; do
    MLRA_THIN_CL=$v timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/cfg2_cl${v}_$i.json 2> /dev/null
    MLRA_THIN_CL=$v timeout 300 python scripts/sweep.py cfg3_1k cfg1 > $O/sweep_cl${v}_$i.jsonl 2>&1
  done
done
timeout 900 python -m pytest tests/test_bench_configs.py -m gpu -x -q -p no:cacheprovider > $O/cfgs.log 2>&1; echo "rc=$?" >> $O/cfgs.log
tail -n 3 $O/parity.log $O/cfgs.log
