# PDL chain + cost-model fix: full gpu suite, A/B with MLRA_PDL=0, probes.
set -x
O=gpurun_out/r02g
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for pdl in 1 0; do
  MLRA_PDL=$pdl timeout 300 python scripts/skinny_probe.py > $O/skinny_pdl$pdl.txt 2>&1
  MLRA_PDL=$pdl timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --no-parity --graph > $O/cfg1_graph_pdl$pdl.json 2> $O/cfg1_graph_pdl$pdl.err
  MLRA_PDL=$pdl timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --no-parity > $O/cfg1_pdl$pdl.json 2> $O/cfg1_pdl$pdl.err
  MLRA_PDL=$pdl timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/cfg2_pdl$pdl.json 2> $O/cfg2_pdl$pdl.err
done
MS=512,1024 timeout 600 python scripts/sk_probe.py > $O/sk_probe.txt 2>&1
