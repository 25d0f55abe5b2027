set -x
O=gpurun_out/r03e
mkdir -p $O
MLRA_PDL=0 timeout 900 python scripts/sweep.py cfg3 cfg4_b3 cfg2 > $O/sweep_nopdl.jsonl 2>&1
timeout 900 python scripts/sweep.py cfg3 cfg4_b3 cfg2 > $O/sweep_pdl.jsonl 2>&1
MLRA_NO_SIDE=1 timeout 900 python scripts/sweep.py cfg3 cfg4_b3 cfg2 > $O/sweep_noside.jsonl 2>&1
