"""bench.py — ModuLoRA fwd+bwd throughput on B200 (driver contract).

Default workload (BASELINE.json configs[1], "cfg2"): the LLaMA-7B MLP pair of
ModuLoRA linears — up 11008x4096 then down 4096x11008 — 3-bit codes, group
128, LoRA rank 16 (alpha 32), 4096 tokens per GPU. One step = forward of both
linears (the down layer consumes the up layer's output), then backward of both
(dX, dA, dB each; dY injected), with (N>1) each layer's LoRA-gradient span
all-reduced (NCCL) as soon as its backward is done. Other BASELINE configs:
--workload cfg1 | cfg3 | cfg4 (cfg3 with --scaling strong splits its 8192
tokens over the ranks). Synthetic data: uniform random codes with RTN-like
grids, A/B ~ N(0, 0.02^2), X/dY ~ N(0, 1) in bf16.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                  [--workload cfg2] [--scaling weak|strong] [--bits B]

--gpus N without a torchrun environment re-launches itself as N ranks
(torch.distributed.run, 127.0.0.1), one per GPU. The timed region is K steps,
each bracketed by CUDA events on the compute stream, with a 512 MiB L2 flush
between steps (outside the events); barrier + synchronize on both sides; the
max over ranks is reported. `e2e` is the same step through the public API
with host (pinned) buffers: X and dY are copied host->device inside the timed
region and the LoRA gradients copied back. `parity` checks one step's outputs
on sampled token rows against an f64 numpy restatement of the layer (bench
code, independent of the library).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "tokens/sec fwd+bwd per ModuLoRA linear (LLaMA-7B/65B shapes), % bf16 TC peak"
_D7, _F7, _D65, _F65 = 4096, 11008, 8192, 22016
WORKLOADS = {
    # name, [(layer, d_out, d_in)], chained?, bits, rank, tokens (per GPU, or global when strong)
    "cfg1": dict(name="cfg1-4096x4096-4bit-r8", layers=[("lin", _D7, _D7)], chain=False, bits=4,
                 rank=8, tokens=512),
    "cfg2": dict(name="cfg2-llama7b-mlp-up+down", layers=[("up", _F7, _D7), ("down", _D7, _F7)],
                 chain=True, bits=3, rank=16, tokens=4096),
    "cfg3": dict(name="cfg3-llama7b-decoder-linear-stack",
                 layers=[("q", _D7, _D7), ("k", _D7, _D7), ("v", _D7, _D7), ("o", _D7, _D7),
                         ("gate", _F7, _D7), ("up", _F7, _D7), ("down", _D7, _F7)],
                 chain=False, bits=3, rank=8, tokens=8192),
    "cfg4": dict(name="cfg4-llama65b-mlp-up+down", layers=[("up", _F65, _D65), ("down", _D65, _F65)],
                 chain=True, bits=3, rank=64, tokens=2048),
}
GROUP, ALPHA = 128, 32.0


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


def workload(args) -> dict:
    w = dict(WORKLOADS[args.workload])
    if args.bits:
        w["bits"] = args.bits
    return w


def tokens_of(w, args, rank, world):
    """(tokens this rank processes, global tokens per step)."""
    if args.scaling == "strong":
        base, extra = divmod(w["tokens"], world)
        return base + (1 if rank < extra else 0), w["tokens"]
    return w["tokens"], w["tokens"] * world


def _config_dict(w, args, world):
    """Identical in both arms (the driver compares them)."""
    return {
        "workload": w["name"],
        "layers": [f"{nm} {o}x{i}" for nm, o, i in w["layers"]],
        "chained": w["chain"], "bits": w["bits"], "group_size": GROUP, "lora_rank": w["rank"],
        "lora_alpha": ALPHA,
        "tokens_per_gpu": w["tokens"] if args.scaling == "weak" else w["tokens"] / world,
        "global_tokens": w["tokens"] * world if args.scaling == "weak" else w["tokens"],
        "parallelism": f"dp{world}" if world > 1 else "single",
        "l2": "flushed between timed steps (512 MiB write, outside the events)",
    }


def step_flops(w, m):
    return sum(4.0 * m * o * i + 6.0 * m * w["rank"] * (o + i) for _, o, i in w["layers"])


def packed_word_count(count: int, bits: int) -> int:
    """bitpack.cpp:64-66 (host arithmetic; numpy only, so the reference arm never
    loads libmlra)."""
    return (count * bits + 31) // 32


def synthetic_codes(rows, cols, bits, group, seed):
    """Uniform random codes in the reference bitstream layout + RTN-like grids
    (numpy only) -> (words u32, scales f32, zeros f32)."""
    rng = np.random.default_rng(seed)
    count = rows * cols
    nw = packed_word_count(count, bits)
    words = rng.integers(0, 2 ** 32, size=nw, dtype=np.uint64).astype(np.uint32)
    tail = nw * 32 - count * bits
    if tail:
        words[-1] &= (1 << (32 - tail)) - 1
    ng = rows * (cols // group)
    # grid of a N(0, 0.02^2) group: range ~ 6 sigma over 2^b - 1 levels
    scales = (0.12 / (2 ** bits - 1) * (0.8 + 0.4 * rng.random(ng))).astype(np.float32)
    zeros = (-0.06 * (0.8 + 0.4 * rng.random(ng))).astype(np.float32)
    return words, scales, zeros


def synthetic_qmatrix(rows, cols, bits, group, seed):
    """synthetic_codes wrapped in the package's host QuantizedMatrix (GPU arm)."""
    from paper_2309_16119_b200 import modulora as M
    words, scales, zeros = synthetic_codes(rows, cols, bits, group, seed)
    return M.QuantizedMatrix(rows, cols, bits, group, M.PackedCodes(bits, rows * cols, words),
                             scales, zeros), words, scales, zeros


# --------------------------------------------------------------------------- parity (numpy)
def _bf16(a):
    """f64 values -> RN f32 -> RN-even bf16, as f64."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def _deq_rows(words, cols, bits, group, sc, z, r0, r1):
    """Rows [r0, r1) of Ŵ = double(s)·c + double(z) (quantize.cpp:130-133) from the
    LSB-first bitstream (bitpack.cpp:25-35); rows word-aligned (every BASELINE shape)."""
    rw = cols * bits // 32
    w = np.asarray(words[r0 * rw:r1 * rw + 1], np.uint64)
    if w.size < (r1 - r0) * rw + 1:
        w = np.append(w, np.uint64(0))
    i = np.arange((r1 - r0) * cols, dtype=np.int64) * bits
    lo, sh = i >> 5, (i & 31).astype(np.uint64)
    c = ((w[lo] | (w[lo + 1] << np.uint64(32))) >> sh) & np.uint64((1 << bits) - 1)
    ng = cols // group
    g = (np.arange(r1 - r0)[:, None] * ng + np.arange(cols)[None, :] // group).ravel()
    s = sc[r0 * ng:r1 * ng].astype(np.float64)[g]
    zz = z[r0 * ng:r1 * ng].astype(np.float64)[g]
    return (s * c.astype(np.float64) + zz).reshape(r1 - r0, cols)


def _rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def parity_check(rec, w, sample=32, seed=7):
    """One step's outputs of every layer against the f64 restatement: sampled
    token rows of Y and dX against the GPU recipe (bf16 Ŵ, bf16(s·xb), bf16 A,
    B; output rounded to bf16) and the exact layer; full dA/dB. Returns
    (ok, worst errors, bars)."""
    bars = {"y_tight": 1e-3, "y_loose": 5e-3, "dx_tight": 1e-3, "dx_loose": 5e-3,
            "dA": 1e-4, "dB": 1e-4}
    worst = {k: 0.0 for k in bars}
    s = ALPHA / w["rank"]
    for (words, sc, z, rows, cols), (x, y, dy, dx, a, b, da, db) in rec:
        m = x.shape[0]
        rs = np.unique(np.random.default_rng(seed).integers(0, m, sample))
        A, B = a.astype(np.float64), b.astype(np.float64)
        x64, dy64 = x.astype(np.float64), dy.astype(np.float64)
        xb, dya = x64 @ B, dy64 @ A
        yb = np.zeros((rs.size, rows))
        ye = np.zeros_like(yb)
        gb = np.zeros((rs.size, cols))
        ge = np.zeros_like(gb)
        for r0 in range(0, rows, 1024):
            r1 = min(rows, r0 + 1024)
            wex = _deq_rows(words, cols, w["bits"], GROUP, sc, z, r0, r1)
            wbf = _bf16(wex)
            yb[:, r0:r1], ye[:, r0:r1] = x64[rs] @ wbf.T, x64[rs] @ wex.T
            gb += dy64[rs, r0:r1] @ wbf
            ge += dy64[rs, r0:r1] @ wex
        e = {"y_tight": _rel(y[rs], _bf16(yb + _bf16(s * xb[rs]) @ _bf16(A).T)),
             "y_loose": _rel(y[rs], ye + s * xb[rs] @ A.T),
             "dx_tight": _rel(dx[rs], _bf16(gb + _bf16(s * dya[rs]) @ _bf16(B).T)),
             "dx_loose": _rel(dx[rs], ge + s * dya[rs] @ B.T),
             "dA": _rel(da, s * dy64.T @ xb), "dB": _rel(db, s * x64.T @ dya)}
        for k, v in e.items():
            worst[k] = max(worst[k], v)
    ok = all(worst[k] <= bars[k] for k in bars)
    return ok, worst, bars


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
def cpu_reference_sample(w, m_per_thread: int, threads: int, seed: int = 1):
    """The reference's own hot path (oracle/_ref: /root/reference/proj/src compiled
    unmodified) on the host cores: `threads` token-sharded single-thread replicas
    of layer_forward + tape backward, for every linear of the workload. Falls back
    to the C oracle port when the reference library is absent. Returns
    (seconds, kind, cores)."""
    from oracle import oracle as orc
    mats = [(synthetic_codes(o, i, w["bits"], GROUP, 11 + k), o, i)
            for k, (_, o, i) in enumerate(w["layers"])]
    if orc.Ref.available():
        t = 0.0
        for (words, sc, z), rows, cols in mats:
            t += orc.Ref.bench_layer(words, rows, cols, w["bits"], GROUP, sc, z, w["rank"], ALPHA,
                                     m_per_thread, threads, seed, strategy=1)
        return t, "reference", threads
    # port: the C restatement, single thread, row-sampled (same algorithm)
    t0 = time.perf_counter()
    for (words, sc, z), rows, cols in mats:
        wt = orc.dequantize(words, rows, cols, w["bits"], GROUP, sc, z)
        a = orc.gaussian(seed, rows, w["rank"], 0.0, 0.02)
        b = orc.gaussian(seed + 1, cols, w["rank"], 0.0, 0.02)
        x = orc.gaussian(seed + 2, m_per_thread, cols)
        g = orc.gaussian(seed + 3, m_per_thread, rows)
        y, xb = orc.layer_forward(wt, a, b, ALPHA, None, x)
        orc.layer_backward(wt, a, b, ALPHA, x, xb, g)
        orc.dequantize(words, rows, cols, w["bits"], GROUP, sc, z)  # bwd re-dequant
    return time.perf_counter() - t0, "port", 1


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    w = workload(args)
    threads = len(os.sched_getaffinity(0)) or 1
    m_pt = 4
    times = []
    for i in range(args.warmup + args.steps):
        t, kind, cores = cpu_reference_sample(w, m_pt, threads, seed=1 + i)
        if i >= args.warmup:
            times.append(t)
    ms = 1e3 * statistics.mean(times)
    value = cores * m_pt / (ms / 1e3)
    sample = (f"{cores} token-sharded single-thread replicas x {m_pt} tokens through every "
              f"linear of the workload (each pass dequantizes the full matrix, as the reference "
              f"does), per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _config_dict(w, args, world),
        "arm": {"strategy": "row (reference RowMaterialize)", "tokens_sampled_per_step": cores * m_pt,
                "host_threads": cores},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": kind,
                         "sample": sample},
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


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args) -> None:
    """--gpus N outside torchrun: re-exec as N ranks (one process per GPU)."""
    backend = os.environ.get("MLRA_DIST_BACKEND", "nccl")
    if args.impl == "ours" and backend == "nccl":
        import torch
        ndev = torch.cuda.device_count()
        if args.gpus > ndev:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but only {ndev} CUDA device(s) visible "
                             "(MLRA_DIST_BACKEND=gloo runs ranks sharing a device, functional only)")
    if backend == "nccl":
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines (nranks per rank)
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


class Workload:
    """The layers of a workload on this rank's device, its inputs and gradient bucket."""

    def __init__(self, w, m, strat, dev, rank):
        import torch
        from paper_2309_16119_b200 import modulora as M
        from paper_2309_16119_b200.dp import GradBucket
        self.w, self.m, self.M = w, m, M
        self.layers, self.host = [], []
        r = w["rank"]
        for i, (nm, rows, cols) in enumerate(w["layers"]):
            q, words, sc, z = synthetic_qmatrix(rows, cols, w["bits"], GROUP, 100 + i)
            g = torch.Generator(device="cpu").manual_seed(200 + i)
            a = (torch.randn(rows, r, generator=g) * 0.02).to(dev)
            b = (torch.randn(cols, r, generator=g) * 0.02).to(dev)
            self.layers.append(M.ModuLoraLayer(nm, M.DeviceQuantizedMatrix(q),
                                               M.LoraAdapter(a, b, r, ALPHA), strategy=strat))
            self.host.append((words, sc, z, rows, cols))
        gen = torch.Generator(device=dev).manual_seed(1234 + rank)
        ins = [w["layers"][0]] if w["chain"] else w["layers"]
        outs = [w["layers"][-1]] if w["chain"] else w["layers"]
        self.xs = [torch.randn(m, i, device=dev, generator=gen).to(torch.bfloat16)
                   for _, _, i in ins]
        self.dys = [torch.randn(m, o, device=dev, generator=gen).to(torch.bfloat16)
                    for _, o, _ in outs]
        self.grads = GradBucket.for_layers(self.layers, dev)
        self.rec = None

    def step(self, xs, dys, before_bwd=None, comm=True, record=False):
        """Forward of every linear, then backward in reverse; each layer's
        gradient span is all-reduced as soon as its backward is done."""
        M, L, gv = self.M, self.layers, self.grads.views
        chain = self.w["chain"]
        acts, xbs, ys = [], [], []
        for i, layer in enumerate(L):
            xin = ys[-1] if (chain and i > 0) else xs[0 if chain else i]
            y, xb = M.layer_forward(layer, xin)
            acts.append(xin)
            xbs.append(xb)
            ys.append(y)
        if before_bwd is not None:
            before_bwd()
        works, upstream, dxs = [], [None] * len(L), [None] * len(L)
        gup = dys[0] if chain else None
        for i in reversed(range(len(L))):
            layer = L[i]
            g = gup if chain else dys[i]
            dx = M.layer_backward(layer, acts[i], xbs[i], g, da=gv[f"{layer.name}.dA"],
                                  db=gv[f"{layer.name}.dB"])
            upstream[i], dxs[i] = g, dx
            if chain:
                gup = dx
            if comm:
                works.append(self.grads.allreduce_async([f"{layer.name}.dA", f"{layer.name}.dB"]))
        for wk in works:
            if wk is not None:
                wk.wait()
        if record:
            def h(t):
                return t.float().cpu().numpy()
            self.rec = [(self.host[i], (h(acts[i]), h(ys[i]), h(upstream[i]), h(dxs[i]),
                                        h(L[i].adapter.a), h(L[i].adapter.b),
                                        h(gv[f"{L[i].name}.dA"]), h(gv[f"{L[i].name}.dB"])))
                        for i in range(len(L))]
        return ys[-1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg2")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="weak: the workload's tokens on every GPU; strong: split over the GPUs")
    ap.add_argument("--bits", type=int, default=0, help="override the workload's code width")
    ap.add_argument("--strategy", default="row", choices=["weight", "row", "matvec"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="replay the step as a captured CUDA graph (default: eager launches)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)  # does not return
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2309_16119_b200 import modulora as M
    from paper_2309_16119_b200._lib import lib

    w = workload(args)
    all_cpus = os.sched_getaffinity(0)
    numa_note = bind_to_gpu_numa_node(local)
    # One rank per GPU. Functional multi-rank runs on a box with fewer GPUs (the
    # 1-GPU dev box) share devices over gloo: MLRA_DIST_BACKEND=gloo.
    ndev = torch.cuda.device_count()
    local = local % ndev if ndev else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = {"backend": None, "nranks": 1}
    if world > 1:
        backend = os.environ.get("MLRA_DIST_BACKEND", "nccl")
        if backend == "nccl":
            # NCCL's own communicator-init lines (nRanks per rank) in the log, also
            # when the driver (not self_launch) started the ranks
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        comm = {"backend": backend, "nranks": dist.get_world_size()}
        print(f"[rank {rank}] {backend} communicator: rank {dist.get_rank()} of "
              f"{dist.get_world_size()} on cuda:{local}", file=sys.stderr, flush=True)
    strat = M.parse_strategy(args.strategy)
    m, global_tokens = tokens_of(w, args, rank, world)
    wl = Workload(w, m, strat, dev, rank)
    grads = wl.grads
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        wl.step(wl.xs, wl.dys)
    torch.cuda.synchronize(dev)
    step = wl.step
    use_graph = args.graph
    if use_graph:
        # The whole fwd+bwd captured once and replayed; the all-reduce stays eager.
        graph = torch.cuda.CUDAGraph()
        c0 = lib().mlra_kernel_launches()
        with torch.cuda.graph(graph):
            wl.step(wl.xs, wl.dys, comm=False)
        graph_kernels = lib().mlra_kernel_launches() - c0
        torch.cuda.synchronize(dev)

        def step(xs, dys, **_):  # noqa: F811  (same inputs as captured)
            graph.replay()
            grads.allreduce()
        for _ in range(2):
            step(wl.xs, wl.dys)
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
            step(wl.xs, wl.dys)
            ev[i][1].record(stream)
        torch.cuda.synchronize(dev)
    launches = lib().mlra_kernel_launches() - launches0
    if use_graph:  # replays launch the captured kernels without touching the host counter
        launches += graph_kernels * args.steps
    total_ms = sum(s.elapsed_time(e) for s, e in ev)
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    ms_per_step = total_ms / args.steps
    value = global_tokens / (ms_per_step / 1e3)

    # ---- parity of one step (same inputs, same calls) on sampled rows, rank 0
    parity = None
    if not args.no_parity:
        wl.step(wl.xs, wl.dys, comm=False, record=rank == 0)
        torch.cuda.synchronize(dev)
        if rank == 0:
            ok, worst, bars = parity_check(wl.rec, w)
            parity = {"status": "ok" if ok else "FAIL", "worst": worst, "bars": bars,
                      "check": "every layer of one step: Y, dX on 32 sampled token rows vs the f64 "
                               "GPU recipe (bf16 out) and the exact f64 layer; dA, dB in full "
                               "(numpy restatement in bench.py)"}
            wl.rec = None

    # ---- dominant kernel: the fused dequant tcgen05 GEMM of the largest linear,
    # timed alone (forward and dX)
    big = max(range(len(wl.layers)), key=lambda i: w["layers"][i][1] * w["layers"][i][2])
    Lb = wl.layers[big]
    ctx = M.LpLinearContext(Lb.weights, strat)
    xbig = torch.randn(m, Lb.d_in(), device=dev).to(torch.bfloat16)
    gbig = torch.randn(m, Lb.d_out(), device=dev).to(torch.bfloat16)
    kt = {}
    for nm, op in (("fwd", lambda: M.lp_forward(ctx, xbig)), ("dx", lambda: M.lp_backward(ctx, gbig))):
        op()
        ts = []
        for _ in range(5):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            op()
            e.record(stream)
            torch.cuda.synchronize(dev)
            ts.append(s.elapsed_time(e))
        kt[nm] = statistics.median(ts)
    k_ms = 0.5 * (kt["fwd"] + kt["dx"])
    gemm_flops = 2.0 * m * Lb.d_in() * Lb.d_out()
    peak_tf, peak_hbm, peak_src = _peaks()
    achieved = gemm_flops / (k_ms / 1e3) / 1e12
    traffic, traffic_split = None, None
    try:  # ncu DRAM bytes of the same kernel at this workload (scripts/traffic.py)
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        if tj.get("workload") == w["name"]:
            traffic = tj.get("qgemm_dram_bytes_per_launch")
            traffic_split = {k: {"dram": tj[k]["dram_read"] + tj[k]["dram_write"],
                                 "algorithmic": tj[k]["alg_read"] + tj[k]["alg_write"]}
                             for k in ("fwd", "dx") if k in tj}
    except Exception:
        pass
    flops = step_flops(w, m)

    # ---- e2e through the public API with host buffers. Every step copies its own
    # inputs (X, dY) from pinned host memory and reads its gradient bucket back.
    # Device input buffers are double-buffered and each input set has its own
    # event: a step's forward waits only for its X, its backward for its dY, so
    # the dY copy (and the next step's copies) overlap compute on the copy
    # engine. The gradient D2H runs on a third stream after the step's last
    # kernel; the next step's backward waits for it before rewriting the bucket.
    n_e2e = max(args.steps, 30)
    xh = [[x.cpu().pin_memory() for x in wl.xs] for _ in range(2)]
    dyh = [[d.cpu().pin_memory() for d in wl.dys] for _ in range(2)]
    gh = torch.empty(grads.flat.numel(), dtype=torch.float32).pin_memory()
    copy_stream, d2h_stream = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    xd = [[torch.empty_like(x) for x in wl.xs] for _ in range(2)]
    dyd = [[torch.empty_like(d) for d in wl.dys] for _ in range(2)]
    ev_x = [torch.cuda.Event() for _ in range(2)]
    ev_dy = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]
    ev_done, ev_read = torch.cuda.Event(), torch.cuda.Event()

    def issue_copy(i):
        sl = i % 2
        with torch.cuda.stream(copy_stream):
            if i >= 2:
                copy_stream.wait_event(ev_free[sl])  # step i-2 finished with this slot
            for d_, h_ in zip(xd[sl], xh[sl]):
                d_.copy_(h_, non_blocking=True)
            ev_x[sl].record(copy_stream)
            for d_, h_ in zip(dyd[sl], dyh[sl]):
                d_.copy_(h_, non_blocking=True)
            ev_dy[sl].record(copy_stream)

    def e2e_run(n):
        issue_copy(0)
        for i in range(n):
            sl = i % 2
            if i + 1 < n:
                issue_copy(i + 1)
            stream.wait_event(ev_x[sl])

            def before_bwd():
                stream.wait_event(ev_dy[sl])
                if i > 0:
                    stream.wait_event(ev_read)  # previous step's gradients read back
            wl.step(xd[sl], dyd[sl], before_bwd=before_bwd)
            ev_free[sl].record(stream)
            ev_done.record(stream)
            with torch.cuda.stream(d2h_stream):
                d2h_stream.wait_event(ev_done)
                gh.copy_(grads.flat, non_blocking=True)
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
    e2e_val = global_tokens / (e2e_ms / 1e3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            os.sched_setaffinity(0, all_cpus)  # the CPU baseline gets every host core
            threads = len(os.sched_getaffinity(0)) or 1
            t, kind, cores = cpu_reference_sample(w, 4, threads)
            cpu = {"value": cores * 4 / t, "unit": "tokens/s", "cores": cores, "kind": kind,
                   "sample": f"{cores} token-sharded replicas x 4 tokens through every linear of "
                             f"the workload ({t:.1f} s; full-matrix dequant per pass, "
                             f"RowMaterialize)"}
            # the reference as designed (one thread): the same 4-token sample
            t1, _, _ = cpu_reference_sample(w, 4, 1, seed=2)
            cpu["single_thread"] = {"value": 4 / t1, "unit": "tokens/s", "cores": 1,
                                    "sample": f"1 thread x 4 tokens ({t1:.1f} s)"}
        except Exception as exc:  # the CPU leg must not kill the GPU number
            cpu = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "unavailable",
                   "sample": repr(exc)[:200]}

    if rank == 0:
        h2d = int(sum(t.numel() * 2 for t in xh[0] + dyh[0]))
        whole_flops = flops * world if args.scaling == "weak" else step_flops(w, global_tokens)
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "bf16",
            "data": f"synthetic (uniform {w['bits']}-bit codes, RTN-like grids; N(0,1) activations)",
            "config": _config_dict(w, args, world),
            "arm": {"strategy": args.strategy,
                    "launch": "cuda-graph replay" if use_graph else "eager",
                    "tokens_this_rank": m},
            "tflops": whole_flops / (ms_per_step / 1e3) / 1e12,
            "pct_bf16_peak": 100.0 * flops / (ms_per_step / 1e3) / 1e12 / peak_tf,
            "roofline": {"bound": "tensor", "kernel": "qgemm2 (fused dequant tcgen05 GEMM)",
                         "layer": f"{w['layers'][big][0]} {Lb.d_out()}x{Lb.d_in()}",
                         "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": achieved / peak_tf, "traffic": traffic, "traffic_by_launch": traffic_split,
                         "frac_sustained": (achieved / _sustained_peak()) if _sustained_peak() else None,
                         "frac_datasheet": achieved / DATASHEET_BF16_TFLOPS,
                         "peak_source": f"{peak_src} bf16 burst (MEASURED_PEAKS.json)",
                         "flops_per_launch": gemm_flops, "launch_ms": k_ms,
                         "launch_ms_fwd": kt["fwd"], "launch_ms_dx": kt["dx"],
                         "gemm_launches_per_step": 2 * len(wl.layers)},
            "parity": parity,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": int(gh.numel() * 4), "ms_per_step": e2e_ms,
                    "steps": n_e2e,
                    "note": "pinned host X/dY copied H2D every step (double-buffered; the forward "
                            "waits for X only, the backward for dY, so copies overlap compute); "
                            "LoRA gradient bucket copied D2H every step on its own stream; the "
                            "region ends after the last D2H; host process " + numa_note},
            "comm": comm,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
