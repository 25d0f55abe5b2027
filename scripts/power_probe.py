"""Dev tool: SM clock / power / throttle reasons while the fused GEMM runs back to back."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml
import torch

from paper_2309_16119_b200 import modulora as M
from scripts.quick_perf import make_layer


def main():
    strat = M.parse_strategy(sys.argv[1] if len(sys.argv) > 1 else "row")
    layer = make_layer(11008, 4096, 3, 16, strat)
    x = torch.randn(4096, 4096, device="cuda").to(torch.bfloat16)
    ctx = M.LpLinearContext(layer.weights, strat)
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    samples, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                            pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
            time.sleep(0.05)

    for _ in range(3):
        M.lp_forward(ctx, x)
    torch.cuda.synchronize()
    th = threading.Thread(target=sample)
    th.start()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 12000
    s.record()
    for _ in range(n):
        M.lp_forward(ctx, x)
    e.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = s.elapsed_time(e) / n
    tail = samples[len(samples) // 3:]
    clk = sorted(c for c, _, _ in tail)[len(tail) // 2]
    pw = sorted(p for _, p, _ in tail)[len(tail) // 2]
    reasons = 0
    for _, _, r in tail:
        reasons |= r
    print(f"{M.strategy_name(strat)}: {ms*1e3:.1f} us/launch = {2*4096*11008*4096/(ms*1e-3)/1e12:.0f} TFLOP/s "
          f"over {n} launches; median SM clock {clk} MHz, power {pw:.0f} W, reasons mask 0x{reasons:x}")


if __name__ == "__main__":
    main()
