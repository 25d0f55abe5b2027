#!/bin/bash
# Round-2 profile captures on the GPU box (one GPU; never multi-rank under ncu).
#   gpurun -- bash scripts/profile_r02.sh [OUT_DIR]
# Every --set full capture is exported on the box (raw + details CSV, SASS source
# page gzipped) and the .ncu-rep removed, so gpurun_out/ stays under its size cap.
set -x
O=${1:-gpurun_out/r02p}
mkdir -p $O
cap() { # name, ncu filter args..., command
  n=$1; shift
  timeout 600 ncu --set full --import-source on --clock-control none -o $O/$n "$@" > $O/$n.log 2>&1
  ncu -i $O/$n.ncu-rep --page raw --csv > $O/$n.raw.csv 2>/dev/null
  ncu -i $O/$n.ncu-rep --page details --csv > $O/$n.details.csv 2>/dev/null
  ncu -i $O/$n.ncu-rep --page source --csv --print-source sass > $O/$n.sass.csv 2>/dev/null
  gzip -f $O/$n.sass.csv; rm -f $O/$n.ncu-rep
}
# 1. launch lists of the bench command (per-launch durations, cold-cache, serialised)
for w in cfg2 cfg1; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$w.csv \
      python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1
done
export REPS=2
# 2. the dominant kernel: cfg2 up layer (11008x4096, 4096 tokens) forward and dX
cap qgemm2_fwd -k regex:qgemm2 -s 1 -c 1 python scripts/ncu_one.py lp_fwd row 11008 4096 3 16 4096
cap qgemm2_dx -k regex:qgemm2 -s 1 -c 1 python scripts/ncu_one.py lp_bwd row 11008 4096 3 16 4096
python scripts/traffic.py $O/qgemm2_fwd.raw.csv $O/qgemm2_dx.raw.csv > $O/traffic.json
# 3. the skinny products of one cfg2 layer pass (prep, rowmma, colmma)
cap thin -k "regex:k_rowmma|k_colmma|k_prep" -s 4 -c 6 python scripts/ncu_one.py layer row 11008 4096 3 16 4096
# 4. K1 materialize at cfg5 (6656x17920 2-bit, bf16 out)
cap k1_cfg5 -k regex:k_materialize -s 1 -c 1 python scripts/ncu_one.py materialize weight 6656 17920 2 8 16
# 5. cfg1 GEMM (4096^2, 512 tokens) under the cost model's choice
cap cfg1_gemm -k regex:qgemm -s 2 -c 1 python scripts/ncu_one.py lp_fwd row 4096 4096 4 8 512
ls -la $O
