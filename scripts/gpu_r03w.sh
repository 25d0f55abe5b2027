# compute-sanitizer over the round-2 code paths (one GPU)
set -x
O=gpurun_out/r03w
mkdir -p $O
CS="compute-sanitizer --error-exitcode 3"
timeout 1500 $CS --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "stream_k or bitwise or arena or golden or layer_llama_shapes" > $O/memcheck_parity.log 2>&1; echo "rc=$?" >> $O/memcheck_parity.log
timeout 1500 $CS --tool memcheck python -m pytest tests/test_e8p.py -m gpu -x -q -p no:cacheprovider -k "not 6656" > $O/memcheck_e8p.log 2>&1; echo "rc=$?" >> $O/memcheck_e8p.log
timeout 1500 $CS --tool memcheck python -m pytest tests/test_bench_configs.py -m gpu -x -q -p no:cacheprovider -k "cfg1" > $O/memcheck_cfg1.log 2>&1; echo "rc=$?" >> $O/memcheck_cfg1.log
timeout 1500 $CS --tool racecheck python -m pytest tests/test_e8p.py -m gpu -x -q -p no:cacheprovider -k "rht" > $O/racecheck_rht.log 2>&1; echo "rc=$?" >> $O/racecheck_rht.log
timeout 1500 $CS --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "bitwise" > $O/racecheck_thin.log 2>&1; echo "rc=$?" >> $O/racecheck_thin.log
for f in $O/*.log; do echo "== $f"; tail -n 4 $f; done
