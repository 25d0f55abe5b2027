set -x
O=gpurun_out/r04a
mkdir -p $O
timeout 300 python scripts/step_timeline.py cfg2 $O/cfg2_trace.json > $O/cfg2_tl.txt 2>&1
timeout 300 python scripts/step_timeline.py cfg1 $O/cfg1_trace.json > $O/cfg1_tl.txt 2>&1
timeout 300 python scripts/step_timeline.py cfg3 $O/cfg3_1k_trace.json 1024 > $O/cfg3_1k_tl.txt 2>&1
gzip -f $O/*.json
tail -5 $O/*_tl.txt
