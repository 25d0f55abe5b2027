for k in 1 2; do
python bench.py --no-cpu-baseline > gpurun_out/e2e_new_$k.log 2>&1
MLRA_E2E_OLD=1 python bench.py --no-cpu-baseline > gpurun_out/e2e_old_$k.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/e2e_*.log")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d["value"]), round(d["e2e"]["value"]), round(d["e2e"]["ms_per_step"],3))
PY
python - <<'PY'
import torch,time
a=torch.empty(64<<20,dtype=torch.uint8).pin_memory(); b=torch.empty(64<<20,dtype=torch.uint8,device="cuda")
for _ in range(3): b.copy_(a,non_blocking=True)
torch.cuda.synchronize(); s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
s.record(); 
for _ in range(10): b.copy_(a,non_blocking=True)
e.record(); torch.cuda.synchronize(); print("H2D GB/s", 10*64*2**20/(s.elapsed_time(e)/1e3)/1e9)
PY
