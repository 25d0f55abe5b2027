# factor conversion with 16-B smem stores; cfg4 (r = 64) A/B fused vs range kernel
set -x
O=gpurun_out/r04h
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "cluster or bitwise or launch_switches or golden" > $O/t.log 2>&1; echo "rc=$?" >> $O/t.log
for i in 1 2; do
  for v in 1 0; do
    MLRA_THIN_CL=$v timeout 300 python scripts/sweep.py cfg4_b3 cfg3_1k cfg1 cfg2 > $O/sweep_cl${v}_$i.jsonl 2>&1
  done
done
tail -n 2 $O/t.log
