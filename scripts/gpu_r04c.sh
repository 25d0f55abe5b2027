# cluster row-product variants (cluster size x ring depth) vs the range kernel
set -x
O=gpurun_out/r04c
mkdir -p $O
MLRA_THIN_CL=0 timeout 300 python scripts/rowmma_probe.py >> $O/probe.jsonl 2>> $O/probe.err
timeout 300 python scripts/rowmma_probe.py >> $O/probe.jsonl 2>> $O/probe.err
for v in c8n4 c8n5 c16n3 c16n5; do
  MLRA_LIB=scripts/var/$v/libmlra.so timeout 300 python scripts/rowmma_probe.py >> $O/probe.jsonl 2>> $O/probe.err
done
for v in c8n5 c16n3; do
  MLRA_LIB=scripts/var/$v/libmlra.so timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/cfg2_$v.json 2> /dev/null
done
timeout 300 python bench.py --no-cpu-baseline --no-parity > $O/cfg2_base.json 2> /dev/null
cat $O/probe.jsonl; tail -3 $O/probe.err
