"""Throughput sweep over BASELINE.json configs on one B200 (reported beside the
headline bench; writes one JSON line per config).

  cfg1  4096x4096, 4-bit g128, r=8, m=512, fwd+bwd
  cfg2  LLaMA-7B MLP up+down, 3-bit, r=16, m=4096 (the bench.py headline)
  cfg3  LLaMA-7B decoder linear stack Q,K,V,O,gate,up,down, 3-bit, r=8, m=8192
  cfg3_1k  the same stack at 1024 tokens (one rank's share of cfg3 strong-scaled over 8 GPUs)
  cfg4  LLaMA-65B up 22016x8192 + down 8192x22016, b in {3,4}, r=64, m=2048 (per GPU of 8)
  cfg5  2-bit 6656x17920 materialize() bandwidth sweep (bf16 and f32 out): the affine
        2-bit format and the black-box "cb2" codebook plugin (hook), plus the cb2 layer
        fwd+bwd through the hook (slabbed hook materialization + tcgen05 GEMM), m=4096
  cfg3_train  the cfg3 stack as a training step (LinearStackTrainer: fwd, bwd, AdamW)
  decoder  the reference's parity-transformer block at LLaMA-7B widths as a device
        training step (model.py: fwd, bwd, AdamW)
  nf4   the lut plugin (NF4, g64) vs the affine 4-bit format at the cfg2 shapes, and
        its materialize() bandwidth at the cfg5 matrix

Timing: CUDA events, 3 warm-up + 10 timed steps, L2 flushed between steps. Each
layer config is timed eager and as a replayed CUDA graph ("launch" key): small
configs (cfg1) are host-launch bound when eager.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import synthetic_qmatrix
from paper_2309_16119_b200 import modulora as M


def layers_for(shapes, bits, r, strat):
    out = []
    for i, (rows, cols) in enumerate(shapes):
        q, *_ = synthetic_qmatrix(rows, cols, bits, 128, 300 + i)
        dq = M.DeviceQuantizedMatrix(q)
        a = torch.randn(rows, r, device="cuda") * 0.02
        b = torch.randn(cols, r, device="cuda") * 0.02
        out.append(M.ModuLoraLayer(f"l{i}", dq, M.LoraAdapter(a, b, r, 32.0), strategy=strat))
    return out


def time_steps(fn, flush, steps=10, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(steps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    return tot / steps


def independent_layers_step(layers, m):
    """fwd+bwd of each linear on its own input (a decoder's linears see
    different inputs; this times the linears, not the glue between them)."""
    xs = [torch.randn(m, L.d_in(), device="cuda").to(torch.bfloat16) for L in layers]
    dys = [torch.randn(m, L.d_out(), device="cuda").to(torch.bfloat16) for L in layers]

    def step():
        for L, x, dy in zip(layers, xs, dys):
            y, xb = M.layer_forward(L, x)
            M.layer_backward(L, x, xb, dy)
    return step


def graphed(fn):
    """Capture fn once (after a warm-up call) and return a replay closure."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    torch.cuda.synchronize()
    return g.replay


def main():
    strat = M.parse_strategy(os.environ.get("STRATEGY", "row"))
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
    try:
        peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                            "MEASURED_PEAKS.json")))
        pk, hbm = float(peaks["bf16_tflops"]), float(peaks["hbm_gbs"])
    except Exception:
        pk, hbm = 1646.4, 6544.3
    cfgs = {
        "cfg1": ([(4096, 4096)], 4, 8, 512),
        "cfg2": ([(11008, 4096), (4096, 11008)], 3, 16, 4096),
        "cfg3": ([(4096, 4096)] * 4 + [(11008, 4096)] * 2 + [(4096, 11008)], 3, 8, 8192),
        # one rank's share of cfg3 strong-scaled over 8 GPUs (8192 / 8 tokens)
        "cfg3_1k": ([(4096, 4096)] * 4 + [(11008, 4096)] * 2 + [(4096, 11008)], 3, 8, 1024),
        "cfg4_b3": ([(22016, 8192), (8192, 22016)], 3, 64, 2048),
        "cfg4_b4": ([(22016, 8192), (8192, 22016)], 4, 64, 2048),
    }
    only = sys.argv[1:]
    for name, (shapes, bits, r, m) in cfgs.items():
        if only and name not in only:
            continue
        layers = layers_for(shapes, bits, r, strat)
        fn = independent_layers_step(layers, m)
        flops = sum(4.0 * m * a * b + 6.0 * m * r * (a + b) for a, b in shapes)
        for launch, f in (("eager", fn), ("cuda-graph", graphed(fn))):
            ms = time_steps(f, flush)
            print(json.dumps({"config": name, "shapes": shapes, "bits": bits, "rank": r,
                              "tokens": m, "strategy": M.strategy_name(strat), "launch": launch,
                              "ms_per_step": ms, "tokens_per_s": m / (ms / 1e3),
                              "tflops": flops / (ms / 1e3) / 1e12,
                              "pct_measured_bf16_peak": 100 * flops / (ms / 1e3) / 1e12 / pk}),
                  flush=True)
        del layers, fn
        torch.cuda.empty_cache()
    if not only or "cfg3_train" in only:
        from paper_2309_16119_b200 import train as T
        shapes, m, r = [(4096, 4096)] * 4 + [(11008, 4096)] * 2 + [(4096, 11008)], 8192, 8
        layers = layers_for(shapes, 3, r, strat)
        tr = T.LinearStackTrainer(layers, T.TrainConfig(lr=1e-4))
        xs = [torch.randn(m, L.d_in(), device="cuda").to(torch.bfloat16) for L in layers]
        dys = [torch.randn(m, L.d_out(), device="cuda").to(torch.bfloat16) for L in layers]
        ms = time_steps(lambda: tr.step(xs, dys, need_dx=True, check_finite=False), flush)
        flops = sum(4.0 * m * a * b + 6.0 * m * r * (a + b) for a, b in shapes)
        print(json.dumps({"config": "cfg3_train", "shapes": shapes, "bits": 3, "rank": r,
                          "tokens": m, "step": "fwd + bwd (with dX) + AdamW over the adapter bucket",
                          "adapter_params": int(tr.params.flat.numel()), "ms_per_step": ms,
                          "tokens_per_s": m / (ms / 1e3), "tflops": flops / (ms / 1e3) / 1e12}),
              flush=True)
        del layers, tr
        torch.cuda.empty_cache()
    if not only or "cfg5" in only:
        q, *_ = synthetic_qmatrix(6656, 17920, 2, 128, 500)
        dq = M.DeviceQuantizedMatrix(q)
        for dt, eb in ((torch.bfloat16, 2), (torch.float32, 4)):
            out = torch.empty(6656, 17920, dtype=dt, device="cuda")
            ms = time_steps(lambda: M.dequantize(dq, dt, out=out), flush)
            nbytes = 6656 * 17920 * (2 / 8 + eb) + 6656 * (17920 // 128) * 8
            print(json.dumps({"config": "cfg5_materialize", "format": "affine", "shape": [6656, 17920],
                              "bits": 2, "out": str(dt), "us": ms * 1e3,
                              "gbs": nbytes / (ms / 1e3) / 1e9,
                              "frac_measured_hbm": nbytes / (ms / 1e3) / 1e9 / hbm}),
                  flush=True)
        # the black-box cb2 plugin (QuIP#-style vector codebook) through its hook
        import numpy as np
        rng = np.random.default_rng(501)
        rows, cols = 6656, 17920
        cbm = M.Cb2Matrix(rows, cols, 128,
                          rng.integers(0, 1 << 16, (rows, cols // 8), dtype=np.uint32).astype(np.uint16),
                          M.default_cb2_codebook(),
                          (0.01 * (0.5 + rng.random((rows, cols // 128)))).astype(np.float32))
        cq = M.Codebook2Quantizer().upload(cbm)
        for dt, eb in ((torch.bfloat16, 2), (torch.float32, 4)):
            out = torch.empty(rows, cols, dtype=dt, device="cuda")
            ms = time_steps(lambda: M.dequantize(cq, dt, out=out), flush)
            nbytes = rows * cols * (2 / 8 + eb) + rows * (cols // 128) * 4 + 8192
            print(json.dumps({"config": "cfg5_materialize", "format": "cb2 plugin (hook)",
                              "shape": [rows, cols], "bits": 2, "out": str(dt), "us": ms * 1e3,
                              "gbs": nbytes / (ms / 1e3) / 1e9,
                              "frac_measured_hbm": nbytes / (ms / 1e3) / 1e9 / hbm}),
                  flush=True)
        del out
        m, r = 4096, 8
        a = torch.randn(rows, r, device="cuda") * 0.02
        b = torch.randn(cols, r, device="cuda") * 0.02
        for sname in ("row", "weight"):
            L = M.ModuLoraLayer("cb2", cq, M.LoraAdapter(a, b, r, 16.0),
                                strategy=M.parse_strategy(sname))
            ms = time_steps(independent_layers_step([L], m), flush)
            flops = 4.0 * m * rows * cols + 6.0 * m * r * (rows + cols)
            print(json.dumps({"config": "cfg5_cb2_layer", "shape": [rows, cols], "rank": r,
                              "tokens": m, "strategy": sname,
                              "ledger_bytes": M.LpLinearContext(cq, L.strategy).ledger_bytes(),
                              "ms_per_step": ms, "tflops": flops / (ms / 1e3) / 1e12}),
                  flush=True)

    if not only or "e8p" in only:
        # the QuIP#-style path at cfg5 shapes: E8P lattice codebook (fused decode in the
        # pair GEMM vs the hook's whole-matrix materialize) and the incoherent layer
        # (block RHT of x / y / dY / dX around the E8P layer)
        import numpy as np
        rows, cols, m, r = 6656, 17920, 4096, 8
        rng = np.random.default_rng(900)
        em = M.E8pMatrix(rows, cols, 128,
                         rng.integers(0, 1 << 16, (rows, cols // 8), dtype=np.uint32).astype(np.uint16),
                         (0.01 * (0.5 + rng.random((rows, cols // 128)))).astype(np.float32))
        eq = M.E8pQuantizer().upload(em)
        for dt, eb in ((torch.bfloat16, 2), (torch.float32, 4)):
            out = torch.empty(rows, cols, dtype=dt, device="cuda")
            ms = time_steps(lambda: M.dequantize(eq, dt, out=out), flush)
            nbytes = rows * cols * (2 / 8 + eb) + rows * (cols // 128) * 4 + 8224
            print(json.dumps({"config": "cfg5_materialize", "format": "e8p plugin (hook)",
                              "shape": [rows, cols], "bits": 2, "out": str(dt), "us": ms * 1e3,
                              "gbs": nbytes / (ms / 1e3) / 1e9,
                              "frac_measured_hbm": nbytes / (ms / 1e3) / 1e9 / hbm}), flush=True)
            del out
        a = torch.randn(rows, r, device="cuda") * 0.02
        b = torch.randn(cols, r, device="cuda") * 0.02
        flops = 4.0 * m * rows * cols + 6.0 * m * r * (rows + cols)
        for sname in ("row", "weight"):
            L = M.ModuLoraLayer("e8p", eq, M.LoraAdapter(a, b, r, 16.0), strategy=M.parse_strategy(sname))
            ms = time_steps(graphed(independent_layers_step([L], m)), flush)
            print(json.dumps({"config": "cfg5_e8p_layer", "shape": [rows, cols], "rank": r,
                              "tokens": m, "strategy": sname, "launch": "cuda-graph",
                              "ledger_bytes": M.LpLinearContext(eq, L.strategy).ledger_bytes(),
                              "ms_per_step": ms, "tflops": flops / (ms / 1e3) / 1e12}), flush=True)
        inc = M.IncoherentLayer(M.ModuLoraLayer("inc", eq, M.LoraAdapter(a, b, r, 16.0)),
                                M.random_signs(rows, 1), M.random_signs(cols, 2), 512)
        x = torch.randn(m, cols, device="cuda").to(torch.bfloat16)
        dy = torch.randn(m, rows, device="cuda").to(torch.bfloat16)

        def inc_step():
            y, saved = inc.forward(x)
            inc.backward(saved, dy)
        ms = time_steps(graphed(inc_step), flush)
        print(json.dumps({"config": "cfg5_e8p_incoherent_layer", "shape": [rows, cols], "rank": r,
                          "tokens": m, "rht_block": 512, "launch": "cuda-graph",
                          "ms_per_step": ms, "tflops": flops / (ms / 1e3) / 1e12}), flush=True)

    if not only or "nf4" in only:
        # the lut plugin (NF4 levels, absmax scale, g64) against the affine 4-bit
        # format at the cfg2 shapes (LLaMA-7B MLP up + down, r=16, m=4096), and its
        # materialize() bandwidth at the cfg5 matrix
        import numpy as np
        rng = np.random.default_rng(700)
        shapes, m, r = [(11008, 4096), (4096, 11008)], 4096, 16

        def lut_dq(rows, cols, bits, group, seed):
            g = np.random.default_rng(seed)
            codes = g.integers(0, 1 << bits, rows * cols, dtype=np.uint32)
            lm = M.LutMatrix(rows, cols, bits, group,
                             M.PackedCodes(bits, rows * cols, M.pack_codes(codes, bits)),
                             M.normal_float_levels(bits),
                             (0.02 * (0.5 + g.random((rows, cols // group)))).astype(np.float32))
            return M.LutQuantizer().upload(lm)

        for fmt in ("nf4", "affine4"):
            layers = []
            for i, (rows, cols) in enumerate(shapes):
                if fmt == "nf4":
                    dq = lut_dq(rows, cols, 4, 64, 710 + i)
                else:
                    q, *_ = synthetic_qmatrix(rows, cols, 4, 64, 720 + i)
                    dq = M.DeviceQuantizedMatrix(q)
                a = torch.randn(rows, r, device="cuda") * 0.02
                b = torch.randn(cols, r, device="cuda") * 0.02
                layers.append(M.ModuLoraLayer(f"{fmt}{i}", dq, M.LoraAdapter(a, b, r, 32.0),
                                              strategy=strat))
            fn = graphed(independent_layers_step(layers, m))
            ms = time_steps(fn, flush)
            flops = sum(4.0 * m * a_ * b_ + 6.0 * m * r * (a_ + b_) for a_, b_ in shapes)
            print(json.dumps({"config": "nf4_mlp", "format": fmt, "shapes": shapes, "bits": 4,
                              "group": 64, "rank": r, "tokens": m, "launch": "cuda-graph",
                              "ms_per_step": ms, "tokens_per_s": m / (ms / 1e3),
                              "tflops": flops / (ms / 1e3) / 1e12,
                              "pct_measured_bf16_peak": 100 * flops / (ms / 1e3) / 1e12 / pk}),
                  flush=True)
            del layers, fn
            torch.cuda.empty_cache()
        rows, cols = 6656, 17920
        dq = lut_dq(rows, cols, 4, 64, 730)
        for dt, eb in ((torch.bfloat16, 2), (torch.float32, 4)):
            out = torch.empty(rows, cols, dtype=dt, device="cuda")
            ms = time_steps(lambda: M.dequantize(dq, dt, out=out), flush)
            nbytes = rows * cols * (4 / 8 + eb) + rows * (cols // 64) * 8
            print(json.dumps({"config": "nf4_materialize", "shape": [rows, cols], "bits": 4,
                              "group": 64, "out": str(dt), "us": ms * 1e3,
                              "gbs": nbytes / (ms / 1e3) / 1e9,
                              "frac_measured_hbm": nbytes / (ms / 1e3) / 1e9 / hbm}),
                  flush=True)
            del out

    if not only or "decoder" in only:
        # the reference's parity-transformer block (model.cpp:226-257) at LLaMA-7B
        # widths as a full training step on the device: 7 quantized linears (3-bit
        # g128, r=16; head to 2 classes) + fp32 glue, backward, AdamW over the
        # adapter bucket. 8 sequences x 512 tokens.
        from paper_2309_16119_b200 import model as Mdl
        from paper_2309_16119_b200 import train as T
        d, dff, B, seq, r = 4096, 11008, 8, 512, 16
        shapes = [(d, d)] * 4 + [(dff, d), (d, dff), (2, d)]
        layers = []
        for i, ((rows, cols), nm) in enumerate(zip(shapes, Mdl.LAYER_NAMES)):
            q, *_ = synthetic_qmatrix(rows, cols, 3, 128, 800 + i)
            a = torch.randn(rows, r, device="cuda") * 0.02
            b = torch.randn(cols, r, device="cuda") * 0.02
            layers.append(M.ModuLoraLayer(nm, M.DeviceQuantizedMatrix(q), M.LoraAdapter(a, b, r, 32.0),
                                          bias=torch.zeros(rows, device="cuda"), strategy=strat))
        tr = Mdl.TransformerTrainer(Mdl.ParityTransformer(layers), T.TrainConfig(lr=1e-4))
        x = torch.randn(B, seq, d, device="cuda")
        y = torch.randint(0, 2, (B,), device="cuda")
        ms = time_steps(lambda: tr.step(x, y, check_finite=False), flush)
        m = B * seq
        lin_flops = sum(4.0 * (m if nm != "head" else B) * a_ * b_ for (a_, b_), nm in zip(shapes, Mdl.LAYER_NAMES))
        print(json.dumps({"config": "decoder_train", "model": "parity_transformer block",
                          "d_model": d, "d_ff": dff, "sequences": B, "seq_len": seq, "bits": 3,
                          "rank": r, "step": "fwd + bwd (dX) + AdamW", "ms_per_step": ms,
                          "tokens_per_s": m / (ms / 1e3),
                          "linear_tflops": lin_flops / (ms / 1e3) / 1e12}), flush=True)
        del layers, tr
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
