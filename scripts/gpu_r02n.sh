set -x
O=gpurun_out/r02n
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_lut.py -m gpu -x -q -p no:cacheprovider -k "materialize or dequant or exact or golden or lut" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python scripts/k1_probe.py > $O/k1.txt 2>&1
timeout 300 python scripts/k1_probe.py > $O/k1b.txt 2>&1
