"""Dev tool: pinned host->device copy bandwidth for the e2e inputs (67 MB per
cfg2 step): one stream vs the copy split over 2 / 4 streams."""
import torch

n = 4096 * 4096
h = [torch.empty(n, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
d = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(2):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for it in range(10):
            for k in range(2):
                chunk = n // ns
                for j, st in enumerate(streams):
                    st.wait_stream(torch.cuda.current_stream()) if it == 0 and k == 0 else None
                    with torch.cuda.stream(st):
                        d[k][j * chunk:(j + 1) * chunk].copy_(h[k][j * chunk:(j + 1) * chunk], non_blocking=True)
        for st in streams:
            torch.cuda.current_stream().wait_stream(st)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        print(f"streams {ns}: {10 * 2 * n * 2 / ms / 1e6:.1f} GB/s")
