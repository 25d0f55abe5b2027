#!/bin/bash
# End-of-round evidence run on one B200: tests, smoke, bench lines (both arms, every
# workload), the sweep, the launch lists and ncu captures; summarised into profiles/
# by scripts/r02_summary.py.   gpurun -- bash scripts/gpu_final.sh [OUT]
set -x
O=${1:-gpurun_out/final}
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for w in cfg1 cfg3 cfg4; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 600 python bench.py --workload cfg1 --graph --no-cpu-baseline > $O/bench_cfg1_graph.json 2> $O/bench_cfg1_graph.err
timeout 1500 python scripts/sweep.py > $O/sweep.jsonl 2> $O/sweep.err
timeout 1500 bash scripts/profile_r02.sh $O/ncu > $O/profile.log 2>&1
du -sh $O
