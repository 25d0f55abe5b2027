set -x
O=gpurun_out/r03b
mkdir -p $O
for i in 1 2; do
  for n in 1 2 4; do
    MLRA_E2E_COPY_STREAMS=$n timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/c${n}_$i.json 2> $O/c${n}_$i.err
  done
done
timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --no-parity > $O/cfg1.json 2> /dev/null
