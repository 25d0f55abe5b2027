set -x
O=gpurun_out/r03v
mkdir -p $O
for i in 1 2; do
  for v in base ns4 ns2 w4; do
    if [ $v = base ]; then L=""; else L="MLRA_LIB=scripts/var/$v/libmlra.so"; fi
    env $L timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/${v}_$i.json 2> /dev/null
    env $L timeout 300 python bench.py --workload cfg1 --graph --no-cpu-baseline --no-parity > $O/cfg1_${v}_$i.json 2> /dev/null
  done
done
