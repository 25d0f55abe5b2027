#!/bin/bash
# Round-2 profile captures on the GPU box (one GPU; never multi-rank under ncu).
#   gpurun -- bash scripts/profile_r02.sh
# Outputs under gpurun_out/r02/; summarised into profiles/ by scripts/ncu_summary.py.
set -x
O=gpurun_out/r02
mkdir -p $O
# 1. launch list of the bench command (per-launch durations, cold-cache, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity > $O/bench_under_ncu.log 2>&1
# 2. the dominant kernel, full sets: cfg2 up layer (11008x4096, 4096 tokens) forward and dX
REPS=2 ncu --set full --import-source on --clock-control none -k regex:qgemm2 -s 1 -c 1 \
    -o $O/qgemm2_fwd python scripts/ncu_one.py lp_fwd row 11008 4096 3 16 4096 > /dev/null 2>&1
REPS=2 ncu --set full --import-source on --clock-control none -k regex:qgemm2 -s 1 -c 1 \
    -o $O/qgemm2_dx python scripts/ncu_one.py lp_bwd row 11008 4096 3 16 4096 > /dev/null 2>&1
# 3. the skinny products of one cfg2 layer pass (rowmma fwd/bwd, colmma dA/dB)
REPS=2 ncu --set full --clock-control none -k "regex:k_rowmma|k_colmma" -s 4 -c 4 \
    -o $O/thin python scripts/ncu_one.py layer row 11008 4096 3 16 4096 > /dev/null 2>&1
# 4. K1 materialize at cfg5 (6656x17920 2-bit, bf16 out)
REPS=2 ncu --set full --clock-control none -k regex:k_materialize -s 1 -c 1 \
    -o $O/k1_cfg5 python scripts/ncu_one.py materialize weight 6656 17920 2 8 16 > /dev/null 2>&1
# 5. cfg1 GEMM (4096^2, 512 tokens) under the cost model's split-K choice
REPS=2 ncu --set full --clock-control none -k regex:qgemm -s 1 -c 1 \
    -o $O/cfg1_split python scripts/ncu_one.py lp_fwd row 4096 4096 4 8 512 > /dev/null 2>&1
ls -la $O
