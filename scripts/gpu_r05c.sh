# step timelines (CUPTI) of cfg1 and cfg2 on the final code
set -x
O=gpurun_out/r05c
mkdir -p $O
timeout 300 python scripts/step_timeline.py cfg1 $O/cfg1_trace.json > $O/cfg1_tl.txt 2>&1
timeout 300 python scripts/step_timeline.py cfg2 $O/cfg2_trace.json > $O/cfg2_tl.txt 2>&1
gzip -f $O/*.json
