set -x
O=gpurun_out/r03n
mkdir -p $O
for pre in 0 1 2 3; do
  MLRA_PRE=$pre MLRA_SK=0 MLRA_LIB=scripts/var/dev/libmlra.so timeout 120 python scripts/trace_mma.py row > $O/trace_pre$pre.txt 2>&1
done
for i in 1 2; do for pre in 0 2 3; do
  MLRA_PRE=$pre timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/pre${pre}_$i.json 2> /dev/null
done; done
