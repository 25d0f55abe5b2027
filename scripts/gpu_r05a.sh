# A/B of the backward side-stream order after the fused row product: default (dA
# early, next to dY·A), MLRA_DA_EARLY=0 (dA after dY·A, filling the dX GEMM's idle
# SMs), MLRA_SIDE_FIRST=1 (dA/dB enqueued before the dX GEMM)
set -x
O=gpurun_out/r05a
mkdir -p $O
for i in 1 2 3; do
  timeout 300 python scripts/sweep.py cfg2 cfg3_1k cfg4_b3 > $O/sweep_default_$i.jsonl 2>&1
  MLRA_DA_EARLY=0 timeout 300 python scripts/sweep.py cfg2 cfg3_1k cfg4_b3 > $O/sweep_late_$i.jsonl 2>&1
  MLRA_SIDE_FIRST=1 timeout 300 python scripts/sweep.py cfg2 cfg3_1k cfg4_b3 > $O/sweep_first_$i.jsonl 2>&1
done
