set -x
O=gpurun_out/r03o
mkdir -p $O
cap() {
  n=$1; shift
  timeout 600 ncu --set full --import-source on --clock-control none -o $O/$n "$@" > $O/$n.log 2>&1
  ncu -i $O/$n.ncu-rep --page raw --csv > $O/$n.raw.csv 2>/dev/null
  rm -f $O/$n.ncu-rep
}
export REPS=2
cap cfg1_gemm -k regex:qgemm -s 1 -c 1 python scripts/ncu_one.py lp_fwd row 4096 4096 4 8 512
cap e8p_gemm -k regex:qgemm2 -s 1 -c 1 python scripts/ncu_one.py e8p_fwd row 6656 17920 2 8 4096
cap rht -k regex:k_rht -s 1 -c 1 python scripts/ncu_one.py rht row 0 17920 2 8 4096
cap thin_cfg1 -k "regex:k_rowmma|k_colmma" -s 3 -c 3 python scripts/ncu_one.py layer row 4096 4096 4 8 512
ls -la $O
