import torch
for dt in (torch.bfloat16, torch.float32):
    out = torch.empty(6656, 17920, dtype=dt, device="cuda")
    src = torch.empty(6656 * 17920 // 8, dtype=torch.uint8, device="cuda")
    for _ in range(3): out.zero_()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): out.zero_()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    print(dt, "zero_ write-only", round(out.numel() * out.element_size() / ms / 1e6, 1), "GB/s")
