# A/B vs the round-1 build (scripts/var/r01, git-ignored) on the same box + launch lists + ncu captures.
set -x
O=gpurun_out/r02b
mkdir -p $O
for i in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --no-parity --steps 20 > $O/new_$i.json 2> $O/new_$i.err
  (cd scripts/var/r01 && timeout 300 python bench.py --no-cpu-baseline --steps 20) > $O/old_$i.json 2> $O/old_$i.err
done
timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --no-parity --graph > $O/cfg1_graph.json 2> $O/cfg1_graph.err
(cd scripts/var/r01 && timeout 400 python scripts/sweep.py cfg1 cfg2 cfg3 cfg4_b3 cfg4_b4) > $O/old_sweep.jsonl 2> $O/old_sweep.err
timeout 400 python scripts/sweep.py cfg1 cfg2 cfg3 cfg4_b3 cfg4_b4 > $O/new_sweep.jsonl 2> $O/new_sweep.err
for w in cfg1 cfg2; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$w.csv \
    python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1
done
cap() { # name, ncu args..., -- command
  n=$1; shift
  timeout 600 ncu --set full --import-source on --clock-control none -o $O/$n "$@" > $O/$n.log 2>&1
  ncu -i $O/$n.ncu-rep --page raw --csv > $O/$n.raw.csv 2>/dev/null
  ncu -i $O/$n.ncu-rep --page details --csv > $O/$n.details.csv 2>/dev/null
  ncu -i $O/$n.ncu-rep --page source --csv --print-source sass > $O/$n.sass.csv 2>/dev/null
  gzip -f $O/$n.sass.csv; rm -f $O/$n.ncu-rep
}
export REPS=2
cap qgemm2_fwd -k regex:qgemm2 -s 1 -c 1 python scripts/ncu_one.py lp_fwd row 11008 4096 3 16 4096
cap qgemm2_dx -k regex:qgemm2 -s 1 -c 1 python scripts/ncu_one.py lp_bwd row 11008 4096 3 16 4096
cap thin -k "regex:k_rowmma|k_colmma|k_prep" -s 4 -c 6 python scripts/ncu_one.py layer row 11008 4096 3 16 4096
cap k1_cfg5 -k regex:k_materialize -s 1 -c 1 python scripts/ncu_one.py materialize weight 6656 17920 2 8 16
cap cfg1_gemm -k regex:qgemm -s 2 -c 2 python scripts/ncu_one.py lp_fwd row 4096 4096 4 8 512
du -sh $O
