# ring depth of the fused row product (k_rowmma_cl): 3 (shipped) vs 4 / 5 stages
set -x
O=gpurun_out/r05i
mkdir -p $O
for v in ns4 ns5; do
  MLRA_LIB=scripts/var/libmlra_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "cluster or chained or bitwise" > $O/t_$v.log 2>&1; echo "rc=$?" >> $O/t_$v.log
  tail -n 2 $O/t_$v.log
done
for i in 1 2 3; do
  timeout 300 python scripts/sweep.py cfg2 cfg3_1k cfg3 > $O/sweep_ns3_$i.jsonl 2>&1
  MLRA_LIB=scripts/var/libmlra_ns4.so timeout 300 python scripts/sweep.py cfg2 cfg3_1k cfg3 > $O/sweep_ns4_$i.jsonl 2>&1
  MLRA_LIB=scripts/var/libmlra_ns5.so timeout 300 python scripts/sweep.py cfg2 cfg3_1k cfg3 > $O/sweep_ns5_$i.jsonl 2>&1
done
for v in ns4 ns5; do
  MLRA_LIB=scripts/var/libmlra_$v.so timeout 120 python - > $O/rowcl_$v.txt 2>&1 <<'PY'
import torch, sys, os
sys.path.insert(0, os.getcwd())
from paper_2309_16119_b200 import modulora as M
from scripts.quick_perf import make_layer
for d_out, d_in, m, r in ((11008, 4096, 4096, 16), (4096, 11008, 4096, 16), (4096, 11008, 1024, 8)):
    L = make_layer(d_out, d_in, 3, r, M.MaterializationStrategy.RowMaterialize)
    x = torch.randn(m, d_in, device="cuda").to(torch.bfloat16)
    for _ in range(3): M.layer_forward(L, x)
    torch.cuda.synchronize()
    print(d_out, d_in, m, r, "ok")
PY
done
