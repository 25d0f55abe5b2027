set -x
O=gpurun_out/r03l
mkdir -p $O
timeout 300 python scripts/h2d_probe.py > $O/h2d.txt 2>&1
for i in 1 2; do
timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --no-parity > $O/cur_$i.json 2> /dev/null
MLRA_DA_EARLY=0 timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --no-parity > $O/noearly_$i.json 2> /dev/null
MLRA_LIB=scripts/var/prearena/libmlra.so timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --no-parity > $O/prearena_$i.json 2> /dev/null
MLRA_LIB=scripts/var/prev/libmlra.so timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --no-parity > $O/prev_$i.json 2> /dev/null
done
timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/cfg2_cur.json 2> /dev/null
MLRA_LIB=scripts/var/prearena/libmlra.so timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/cfg2_prearena.json 2> /dev/null
