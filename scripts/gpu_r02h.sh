# PDL A/B (dX GEMM with side-stream dA/dB launched classically)
set -x
O=gpurun_out/r02h
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_bench_configs.py tests/test_model.py -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for i in 1 2 3; do for pdl in 1 0; do
  MLRA_PDL=$pdl timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/cfg2_pdl${pdl}_$i.json 2> /dev/null
  MLRA_PDL=$pdl timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --no-parity --graph > $O/cfg1g_pdl${pdl}_$i.json 2> /dev/null
  MLRA_PDL=$pdl timeout 300 python bench.py --workload cfg3 --scaling strong --gpus 1 --no-cpu-baseline --no-parity > $O/cfg3_pdl${pdl}_$i.json 2> /dev/null
done; done
for pdl in 1 0; do MLRA_PDL=$pdl timeout 300 python scripts/skinny_probe.py > $O/skinny_pdl$pdl.txt 2>&1; done
