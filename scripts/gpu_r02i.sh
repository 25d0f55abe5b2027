set -x
O=gpurun_out/r02i
mkdir -p $O
timeout 1500 python scripts/sweep.py > $O/sweep.jsonl 2> $O/sweep.err
timeout 1200 bash scripts/profile_r02.sh gpurun_out/r02p > $O/profile.log 2>&1
du -sh gpurun_out/r02p
