"""bench.py — ModuLoRA fwd+bwd throughput on B200 (driver contract).

Workload (BASELINE.json configs[1], "cfg2"): the LLaMA-7B MLP pair of
ModuLoRA linears — up 11008x4096 then down 4096x11008 — 3-bit codes, group
128, LoRA rank 16 (alpha 32), 4096 tokens per GPU. One step = forward of both
linears (the down layer consumes the up layer's output), then backward of both
(dX, dA, dB each; dY injected), then (N>1) one NCCL all-reduce of the LoRA
gradient bucket. Synthetic data: uniform random codes with RTN-like grids,
A/B ~ N(0, 0.02^2), X/dY ~ N(0, 1) in bf16.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

The timed region is K steps, each bracketed by CUDA events on the compute
stream, with a 512 MiB L2 flush between steps (outside the events); barrier +
synchronize on both sides; the max over ranks is reported. `e2e` is the same
step through the public API with host (pinned) buffers: X and dY are copied
host->device inside the timed region and the LoRA gradients copied back.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CFG = dict(name="cfg2-llama7b-mlp-up+down", m=4096, d_model=4096, d_ff=11008, bits=3, group=128,
           rank=16, alpha=32.0)
METRIC = "tokens/sec fwd+bwd per ModuLoRA linear (LLaMA-7B/65B shapes), % bf16 TC peak"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["bf16_tflops"]), float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 1590.0, 6650.0, "fallback"


def _sustained_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops_sustained"])
    except Exception:
        return None


DATASHEET_BF16_TFLOPS = 2250.0  # dense bf16 per B200 (the 4500 figure is 2:4 sparse)


def _config_dict(strategy: str, n: int):
    return {
        "workload": CFG["name"],
        "layers": [f"up {CFG['d_ff']}x{CFG['d_model']}", f"down {CFG['d_model']}x{CFG['d_ff']}"],
        "bits": CFG["bits"], "group_size": CFG["group"], "lora_rank": CFG["rank"],
        "lora_alpha": CFG["alpha"], "tokens_per_gpu": CFG["m"], "global_tokens": CFG["m"] * n,
        "strategy": strategy, "parallelism": f"dp{n}" if n > 1 else "single",
        "l2": "flushed between timed steps (512 MiB write, outside the events)",
    }


def synthetic_qmatrix(rows, cols, bits, group, seed):
    """Uniform random codes in the reference bitstream layout + RTN-like grids."""
    from paper_2309_16119_b200 import modulora as M
    rng = np.random.default_rng(seed)
    count = rows * cols
    nw = M.packed_word_count(count, bits)
    words = rng.integers(0, 2 ** 32, size=nw, dtype=np.uint64).astype(np.uint32)
    tail = nw * 32 - count * bits
    if tail:
        words[-1] &= (1 << (32 - tail)) - 1
    ng = rows * (cols // group)
    # grid of a N(0, 0.02^2) group: range ~ 6 sigma over 2^b - 1 levels
    scales = (0.12 / (2 ** bits - 1) * (0.8 + 0.4 * rng.random(ng))).astype(np.float32)
    zeros = (-0.06 * (0.8 + 0.4 * rng.random(ng))).astype(np.float32)
    return M.QuantizedMatrix(rows, cols, bits, group, M.PackedCodes(bits, count, words), scales,
                             zeros), words, scales, zeros


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clock + throttle reasons
    during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        "display_clock_setting": 0x100,
    }

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                mask = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for k, bit in self.REASONS.items():
                    if mask & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self._ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._ok:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons)}


# --------------------------------------------------------------------------- CPU legs
def cpu_reference_sample(m_per_thread: int, threads: int, seed: int = 1):
    """The reference's own hot path (oracle/_ref: /root/reference/proj/src compiled
    unmodified) on the host cores: `threads` token-sharded single-thread replicas
    of layer_forward + tape backward, for both linears of the workload. Falls
    back to the C oracle port when the reference library is absent."""
    sys.path.insert(0, ROOT)
    from oracle import oracle as orc
    up = synthetic_qmatrix(CFG["d_ff"], CFG["d_model"], CFG["bits"], CFG["group"], 11)
    down = synthetic_qmatrix(CFG["d_model"], CFG["d_ff"], CFG["bits"], CFG["group"], 12)
    if orc.Ref.available():
        t = 0.0
        for (q, words, sc, z) in (up, down):
            t += orc.Ref.bench_layer(words, q.rows, q.cols, q.bits, q.group_size, sc, z,
                                     CFG["rank"], CFG["alpha"], m_per_thread, threads, seed,
                                     strategy=1)
        return t, "reference", threads
    # port: the C restatement, single thread, row-sampled (same algorithm)
    t0 = time.perf_counter()
    for (q, words, sc, z) in (up, down):
        w = orc.dequantize(words, q.rows, q.cols, q.bits, q.group_size, sc, z)
        a = orc.gaussian(seed, q.rows, CFG["rank"], 0.0, 0.02)
        b = orc.gaussian(seed + 1, q.cols, CFG["rank"], 0.0, 0.02)
        x = orc.gaussian(seed + 2, m_per_thread, q.cols)
        g = orc.gaussian(seed + 3, m_per_thread, q.rows)
        y, xb = orc.layer_forward(w, a, b, CFG["alpha"], None, x)
        orc.layer_backward(w, a, b, CFG["alpha"], x, xb, g)
        orc.dequantize(words, q.rows, q.cols, q.bits, q.group_size, sc, z)  # bwd re-dequant
    return time.perf_counter() - t0, "port", 1


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    threads = len(os.sched_getaffinity(0)) or 1
    m_pt = 4
    times = []
    for i in range(args.warmup + args.steps):
        t, kind, cores = cpu_reference_sample(m_pt, threads, seed=1 + i)
        if i >= args.warmup:
            times.append(t)
    ms = 1e3 * statistics.mean(times)
    value = cores * m_pt / (ms / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _config_dict("row (reference RowMaterialize)", 1),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": kind,
                         "sample": f"{cores} replicas x {m_pt} tokens of the up+down pair "
                                   f"(full 11008x4096 dequant per pass), per step"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- GPU arm
def bind_to_gpu_numa_node(device_index: int) -> str:
    """Pin this process to the CPU cores NVML reports as closest to the GPU, so
    pinned host buffers (first touch) land on the GPU's NUMA node and the e2e
    host<->device copies take the local PCIe path. Returns a note."""
    if os.environ.get("MLRA_NO_NUMA_BIND"):
        return "not bound (MLRA_NO_NUMA_BIND)"
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 64)
        cpus = {64 * w + b for w, mask in enumerate(words) for b in range(64) if mask >> b & 1}
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
            return f"bound to {len(cpus)} GPU-local cores"
    except Exception as e:  # best effort: no NVML / affinity API
        return f"not bound ({type(e).__name__})"
    return "not bound"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--strategy", default="row", choices=["weight", "row", "matvec"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="replay the step as a captured CUDA graph (default: eager launches; "
                         "measured equal at cfg2)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2309_16119_b200 import modulora as M
    from paper_2309_16119_b200._lib import lib

    all_cpus = os.sched_getaffinity(0)
    numa_note = bind_to_gpu_numa_node(local)
    # One rank per GPU. Functional multi-rank runs on a box with fewer GPUs (the
    # 1-GPU dev box) may share devices and use gloo: MLRA_DIST_BACKEND=gloo.
    ndev = torch.cuda.device_count()
    local = local % ndev if ndev else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("MLRA_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    strat = M.parse_strategy(args.strategy)
    m, r = CFG["m"], CFG["rank"]

    layers = []
    for i, (rows, cols) in enumerate(((CFG["d_ff"], CFG["d_model"]), (CFG["d_model"], CFG["d_ff"]))):
        q, *_ = synthetic_qmatrix(rows, cols, CFG["bits"], CFG["group"], 100 + i)
        dq = M.DeviceQuantizedMatrix(q)
        g = torch.Generator(device="cpu").manual_seed(200 + i)
        a = (torch.randn(rows, r, generator=g) * 0.02).to(dev)
        b = (torch.randn(cols, r, generator=g) * 0.02).to(dev)
        layers.append(M.ModuLoraLayer(f"l{i}", dq, M.LoraAdapter(a, b, r, CFG["alpha"]), strategy=strat))
    up, down = layers
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    x = torch.randn(m, CFG["d_model"], device=dev, generator=gen).to(torch.bfloat16)
    dy2 = torch.randn(m, CFG["d_model"], device=dev, generator=gen).to(torch.bfloat16)
    # one flat LoRA-gradient bucket: [dA_up | dB_up | dA_down | dB_down] -> one all-reduce
    from paper_2309_16119_b200.dp import GradBucket
    grads = GradBucket.for_layers([up, down], dev)
    bucket = grads.flat
    da_up, db_up = grads.views["l0.dA"], grads.views["l0.dB"]
    da_dn, db_dn = grads.views["l1.dA"], grads.views["l1.dB"]

    def step(xin, dyin):
        y1, xb1 = M.layer_forward(up, xin)
        y2, xb2 = M.layer_forward(down, y1)
        dx2 = M.layer_backward(down, y1, xb2, dyin, da=da_dn, db=db_dn)
        # the down layer's gradients all-reduce (NCCL) while the up layer's backward runs
        w_dn = grads.allreduce_async(["l1.dA", "l1.dB"])
        M.layer_backward(up, xin, xb1, dx2, da=da_up, db=db_up)
        w_up = grads.allreduce_async(["l0.dA", "l0.dB"])
        for w in (w_dn, w_up):
            if w is not None:
                w.wait()
        return y2

    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def compute(xin, dyin):
        y1, xb1 = M.layer_forward(up, xin)
        y2, xb2 = M.layer_forward(down, y1)
        dx2 = M.layer_backward(down, y1, xb2, dyin, da=da_dn, db=db_dn)
        M.layer_backward(up, xin, xb1, dx2, da=da_up, db=db_up)

    for _ in range(args.warmup):
        step(x, dy2)
    torch.cuda.synchronize(dev)
    use_graph = args.graph
    if use_graph:
        # The whole fwd+bwd of the layer pair (~20 kernels, stream-ordered scratch,
        # side-stream fork/join) captured once and replayed: no per-launch host
        # overhead or inter-kernel gaps. The NCCL all-reduce stays eager.
        graph = torch.cuda.CUDAGraph()
        c0 = lib().mlra_kernel_launches()
        with torch.cuda.graph(graph):
            compute(x, dy2)
        graph_kernels = lib().mlra_kernel_launches() - c0  # libmlra kernels in one replay
        torch.cuda.synchronize(dev)

        def step(xin, dyin):  # noqa: F811  (same inputs as captured)
            graph.replay()
            grads.allreduce()
        for _ in range(2):
            step(x, dy2)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches0 = lib().mlra_kernel_launches()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            step(x, dy2)
            ev[i][1].record(stream)
        torch.cuda.synchronize(dev)
    launches = lib().mlra_kernel_launches() - launches0
    if use_graph:  # replays launch the captured kernels without touching the host counter
        launches += graph_kernels * args.steps
    step_ms = [s.elapsed_time(e) for s, e in ev]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    ms_per_step = total_ms / args.steps
    value = world * m / (ms_per_step / 1e3)

    # ---- dominant kernel: the fused dequant tcgen05 GEMM, timed alone (4 launches/step,
    # identical FLOPs 2·m·d_ff·d_model each: fwd up, fwd down, dX down, dX up)
    ctx_up = M.LpLinearContext(up.weights, strat)
    ctx_dn = M.LpLinearContext(down.weights, strat)
    y1 = M.layer_forward(up, x)[0]
    ops = [lambda: M.lp_forward(ctx_up, x), lambda: M.lp_forward(ctx_dn, y1),
           lambda: M.lp_backward(ctx_dn, dy2), lambda: M.lp_backward(ctx_up, y1)]
    kt = []
    for op in ops:
        op()
        for _ in range(3):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            op()
            e.record(stream)
            torch.cuda.synchronize(dev)
            kt.append(s.elapsed_time(e))
    k_ms = statistics.mean(kt)
    gemm_flops = 2.0 * m * CFG["d_ff"] * CFG["d_model"]
    peak_tf, peak_hbm, peak_src = _peaks()
    achieved = gemm_flops / (k_ms / 1e3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get("qgemm_dram_bytes_per_launch")
    except Exception:
        pass
    step_flops = 2 * (4.0 * m * CFG["d_ff"] * CFG["d_model"] + 6.0 * m * r * (CFG["d_ff"] + CFG["d_model"]))

    # ---- e2e through the public API with host buffers. Every step copies its own
    # X and dY from pinned host memory and reads its gradient bucket back. The
    # device input buffers are double-buffered and each input has its own event:
    # a step's forward waits only for its X, its backward for its dY, so dY's
    # copy (and the next step's copies) overlap compute on the copy engine. The
    # gradient D2H runs on a third stream (the other copy direction) after the
    # step's last kernel, and the next step's backward waits for it before
    # rewriting the bucket. The first step's copies are inside the timed region;
    # the final synchronize covers the last D2H.
    # a steady-state stream of steps: at least 30, so the first step's exposed
    # copy (nothing earlier to overlap it with) is a startup cost, not a third
    # of the number; still every step pays its own H2D + D2H inside the region
    n_e2e = max(args.steps, 30)
    xh = [x.cpu().pin_memory() for _ in range(2)]
    dyh = [dy2.cpu().pin_memory() for _ in range(2)]
    gh = torch.empty(bucket.numel(), dtype=torch.float32).pin_memory()
    copy_stream = torch.cuda.Stream(dev)
    d2h_stream = torch.cuda.Stream(dev)
    xd = [torch.empty_like(x) for _ in range(2)]
    dyd = [torch.empty_like(dy2) for _ in range(2)]
    ev_x = [torch.cuda.Event() for _ in range(2)]
    ev_dy = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]
    ev_done, ev_read = torch.cuda.Event(), torch.cuda.Event()

    def issue_copy(i):
        sl = i % 2
        with torch.cuda.stream(copy_stream):
            if i >= 2:
                copy_stream.wait_event(ev_free[sl])  # step i-2 finished with this slot
            xd[sl].copy_(xh[sl], non_blocking=True)
            ev_x[sl].record(copy_stream)
            dyd[sl].copy_(dyh[sl], non_blocking=True)
            ev_dy[sl].record(copy_stream)

    def e2e_run(n):
        issue_copy(0)
        for i in range(n):
            sl = i % 2
            if i + 1 < n:
                issue_copy(i + 1)
            stream.wait_event(ev_x[sl])
            y1, xb1 = M.layer_forward(up, xd[sl])
            y2, xb2 = M.layer_forward(down, y1)
            stream.wait_event(ev_dy[sl])
            if i > 0:
                stream.wait_event(ev_read)  # previous step's gradients read back
            dx2 = M.layer_backward(down, y1, xb2, dyd[sl], da=da_dn, db=db_dn)
            w_dn = grads.allreduce_async(["l1.dA", "l1.dB"])
            M.layer_backward(up, xd[sl], xb1, dx2, da=da_up, db=db_up)
            w_up = grads.allreduce_async(["l0.dA", "l0.dB"])
            for w in (w_dn, w_up):
                if w is not None:
                    w.wait()
            ev_free[sl].record(stream)
            ev_done.record(stream)
            with torch.cuda.stream(d2h_stream):
                d2h_stream.wait_event(ev_done)
                gh.copy_(bucket, non_blocking=True)
                ev_read.record(d2h_stream)

    e2e_run(3)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    e2e_run(n_e2e)
    stream.wait_event(ev_read)  # the last step's gradient read-back is inside the region
    e.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = s.elapsed_time(e) / n_e2e
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_val = world * m / (e2e_ms / 1e3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            os.sched_setaffinity(0, all_cpus)  # the CPU baseline gets every host core
            threads = len(os.sched_getaffinity(0)) or 1
            t, kind, cores = cpu_reference_sample(4, threads)
            cpu = {"value": cores * 4 / t, "unit": "tokens/s", "cores": cores, "kind": kind,
                   "sample": f"{cores} token-sharded replicas x 4 tokens of the up+down pair "
                             f"({t:.1f} s; full-matrix dequant per pass, RowMaterialize)"}
            # the reference as designed (one thread): the same 4-token sample
            t1, _, _ = cpu_reference_sample(4, 1, seed=2)
            cpu["single_thread"] = {"value": 4 / t1, "unit": "tokens/s", "cores": 1,
                                    "sample": f"1 thread x 4 tokens ({t1:.1f} s)"}
        except Exception as exc:  # the CPU leg must not kill the GPU number
            cpu = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "unavailable",
                   "sample": repr(exc)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (uniform 3-bit codes, RTN-like grids; N(0,1) activations)",
            "config": dict(_config_dict(args.strategy, world),
                           launch="cuda-graph replay" if use_graph else "eager"),
            "tflops": step_flops / (ms_per_step / 1e3) / 1e12,
            "pct_bf16_peak": 100.0 * step_flops / (ms_per_step / 1e3) / 1e12 / peak_tf,
            "roofline": {"bound": "tensor", "kernel": "qgemm (fused dequant tcgen05 GEMM)",
                         "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": achieved / peak_tf, "traffic": traffic,
                         "frac_sustained": (achieved / _sustained_peak()) if _sustained_peak() else None,
                         "frac_datasheet": achieved / DATASHEET_BF16_TFLOPS,
                         "peak_source": f"{peak_src} bf16 burst (MEASURED_PEAKS.json)",
                         "flops_per_launch": gemm_flops, "launch_ms": k_ms,
                         "launches_per_step": 4,
                         "share_of_step": 4 * k_ms / ms_per_step},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "tokens/s",
                    "h2d_bytes_per_step": int(xh[0].numel() * 2 + dyh[0].numel() * 2),
                    "d2h_bytes_per_step": int(gh.numel() * 4), "ms_per_step": e2e_ms,
                    "steps": n_e2e,
                    "note": "pinned host X/dY copied H2D every step (double-buffered; the forward "
                            "waits for X only, the backward for dY, so copies overlap compute); "
                            "LoRA gradient bucket copied D2H every step on its own stream; the "
                            "region ends after the last D2H; host process " + numa_note},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
