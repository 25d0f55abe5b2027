"""GPU parity at the BASELINE configs the bench and the sweep time.

Every config of BASELINE.json with a ModuLoRA fwd+bwd is run here at its full
shape and token count, on the bench's own synthetic weights, through the same
calls the bench makes, under every GEMM schedule that shape can take:

  * cfg2  LLaMA-7B MLP up 11008x4096 -> down 4096x11008, 3-bit g128, r=16,
          m=4096 (the bench.py headline chain: 344 pair tiles = ~4.6 whole tiles
          per CTA pair, dX with 172 k-blocks per tile);
  * cfg4  LLaMA-65B up 22016x8192 -> down 8192x22016, b in {3, 4}, r=64 (one
          full 64-wide LoRA k-block), m=2048 tokens per GPU;
  * cfg3  the LLaMA-7B decoder linear stack (Q,K,V,O 4096², gate/up
          11008x4096, down 4096x11008), 3-bit, r=8, 8192 tokens;
  * cfg5  the cb2 (QuIP#-style 2-bit codebook) plugin layer 6656x17920, r=8,
          m=4096, fused decode and through the hook;
  * a multi-wave 4096² m=4096 case under the 1-CTA and the pair kernel.

Schedules: the default plan, MLRA_SK=0 (whole tiles strided over the pairs;
several tiles per pair with the accumulator ping-pong) and MLRA_SK=1 (stream-K
split tiles with the ordered fix-up). Checks (tests/gpu_util.check_layer_pass):
xb, dA, dB in full against f64 on the same inputs; Y and dX on one seeded row
per 128-token sub-tile against the f64 GPU recipe (<= 1e-4) and the exact f64
layer (<= 4e-3). The bf16-output epilogue (paired-row stores) must equal the
RN-bf16 of the fp32-output epilogue bit for bit (same MMA order).

Reference products matched: lp_forward / lp_backward
(proj/src/lowprec_linear.cpp:150-247), the adapter records of layer_forward
(proj/src/lora.cpp:67-71) and their backward rules (autodiff.cpp:145-193);
dense-oracle check as proj/tests/test_lora.cpp:123-150.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2309_16119_b200 import modulora as M
from tests.conftest import rel_fro
from tests.gpu_util import check_layer_pass, deq_products, f64, synthetic, to_bf16_dev

pytestmark = pytest.mark.gpu

ROW = M.MaterializationStrategy.RowMaterialize
SCHEDULES = {"default": {}, "whole": {"MLRA_SK": "0", "MLRA_GEMM": "2"},
             "streamk": {"MLRA_SK": "1", "MLRA_GEMM": "2"},
             "splitk": {"MLRA_SK": "4", "MLRA_GEMM": "2"},
             "splitk256": {"MLRA_SK": "5", "MLRA_GEMM": "2"}}


def _setenv(monkeypatch, env):
    for k in ("MLRA_SK", "MLRA_GEMM"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)


class Lin:
    """One synthetic ModuLoRA linear of a config + its host-side oracle inputs."""

    def __init__(self, rows, cols, bits, r, seed, alpha=32.0, bias=False, strategy=ROW):
        q, self.words, self.sc, self.z = synthetic(rows, cols, bits, 128, seed)
        self.rows, self.cols, self.bits, self.alpha = rows, cols, bits, alpha
        rng = np.random.default_rng(seed + 1)
        self.a32 = (0.02 * rng.standard_normal((rows, r))).astype(np.float32)
        self.b32 = (0.02 * rng.standard_normal((cols, r))).astype(np.float32)
        self.bias32 = (0.1 * rng.standard_normal(rows)).astype(np.float32) if bias else None
        self.layer = M.ModuLoraLayer(
            f"l{seed}", M.DeviceQuantizedMatrix(q),
            M.LoraAdapter(torch.from_numpy(self.a32).cuda(), torch.from_numpy(self.b32).cuda(), r,
                          alpha),
            bias=None if self.bias32 is None else torch.from_numpy(self.bias32).cuda(),
            strategy=strategy)

    def deq(self, xr, gr):
        return deq_products(self.words, self.rows, self.cols, self.bits, 128, self.sc, self.z, xr,
                            gr)

    def run(self, x, dy):
        """fwd + bwd with fp32 outputs, and again with bf16 outputs: the bf16
        epilogue must be the RN-bf16 of the fp32 one (same accumulation)."""
        L = self.layer
        y, xb = M.layer_forward(L, x, out_dtype=torch.float32)
        y16, xb16 = M.layer_forward(L, x, out_dtype=torch.bfloat16)
        assert torch.equal(y16, y.to(torch.bfloat16)), "bf16 epilogue != RN(fp32 epilogue)"
        assert torch.equal(xb16, xb)
        dx16 = M.layer_backward(L, x, xb, dy, dx_dtype=torch.bfloat16)
        da16, db16 = (t.clone() for t in M.grads_of_adapter(L))
        dx = M.layer_backward(L, x, xb, dy, dx_dtype=torch.float32)
        da, db = M.grads_of_adapter(L)
        assert torch.equal(dx16, dx.to(torch.bfloat16)), "bf16 dX epilogue != RN(fp32 epilogue)"
        # dA / dB: ordered (deterministic) reductions -> bitwise equal across runs
        assert torch.equal(da16, da) and torch.equal(db16, db)
        return y, y16, xb, dx, dx16, da, db

    def check(self, x, dy, out, what):
        y, _, xb, dx, _, da, db = out
        return check_layer_pass(self.deq, self.a32, self.b32, self.alpha, f64(x), f64(dy), y, xb,
                                dx, da, db, bias32=self.bias32, what=what)


def _act(seed, m, d):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return torch.randn(m, d, generator=g).to(torch.bfloat16).cuda()


@pytest.mark.parametrize("sched", list(SCHEDULES))
def test_cfg2_mlp_chain(sched, monkeypatch):
    """bench.py's step: up fwd -> down fwd (on up's bf16 output) -> down bwd ->
    up bwd (on down's bf16 dX), 4096 tokens."""
    _setenv(monkeypatch, SCHEDULES[sched])
    m, r = 4096, 16
    up = Lin(11008, 4096, 3, r, seed=100)
    down = Lin(4096, 11008, 3, r, seed=101, bias=True)
    x = _act(1, m, 4096)
    dy2 = _act(2, m, 4096)
    o_up_fwd = M.layer_forward(up.layer, x)  # bf16 y1 feeds the down layer, as in bench.py
    y1 = o_up_fwd[0]
    o_dn = down.run(y1, dy2)
    dx2 = o_dn[4]  # bf16 dX of the down layer is the up layer's upstream gradient
    o_up = up.run(x, dx2)
    assert torch.equal(o_up[1], y1)
    down.check(y1, dy2, o_dn, f"cfg2 down [{sched}]")
    up.check(x, dx2, o_up, f"cfg2 up [{sched}]")


@pytest.mark.parametrize("bits", [3, 4])
@pytest.mark.parametrize("sched", ["default", "whole"])
def test_cfg4_llama65b_pair(bits, sched, monkeypatch):
    """LLaMA-65B MLP up 22016x8192 -> down 8192x22016, r=64, 2048 tokens per GPU."""
    _setenv(monkeypatch, SCHEDULES[sched])
    m, r = 2048, 64
    up = Lin(22016, 8192, bits, r, seed=200 + bits)
    down = Lin(8192, 22016, bits, r, seed=210 + bits)
    x = _act(3, m, 8192)
    dy2 = _act(4, m, 8192)
    y1 = M.layer_forward(up.layer, x)[0]
    o_dn = down.run(y1, dy2)
    o_up = up.run(x, o_dn[4])
    down.check(y1, dy2, o_dn, f"cfg4 b{bits} down [{sched}]")
    up.check(x, o_dn[4], o_up, f"cfg4 b{bits} up [{sched}]")


def test_cfg3_decoder_stack():
    """The seven LLaMA-7B decoder linears at 8192 tokens, 3-bit, r=8 (each on its
    own seeded input, as scripts/sweep.py times them)."""
    m, r = 8192, 8
    shapes = [(4096, 4096)] * 4 + [(11008, 4096)] * 2 + [(4096, 11008)]
    names = ["q", "k", "v", "o", "gate", "up", "down"]
    for i, ((rows, cols), nm) in enumerate(zip(shapes, names)):
        lin = Lin(rows, cols, 3, r, seed=300 + i)
        x = _act(30 + i, m, cols)
        dy = _act(40 + i, m, rows)
        lin.check(x, dy, lin.run(x, dy), f"cfg3 {nm}")
        del lin
        torch.cuda.empty_cache()


@pytest.mark.parametrize("gemm", ["1", "2", "3"])
def test_multi_wave_whole_tiles(gemm, monkeypatch):
    """more tiles than CTAs (4096² at m=4096: 128 pair tiles over 74
    pairs, 256 1-CTA tiles over 148 CTAs) with whole tiles, LoRA and bias; the
    stream-K result of the pair kernel agrees to fp32 order."""
    _setenv(monkeypatch, {"MLRA_SK": "0", "MLRA_GEMM": gemm})
    lin = Lin(4096, 4096, 4, 16, seed=400, bias=True)
    x = _act(50, 4096, 4096)
    dy = _act(51, 4096, 4096)
    out = lin.run(x, dy)
    lin.check(x, dy, out, f"multi-wave gemm={gemm}")
    _setenv(monkeypatch, {"MLRA_SK": "1", "MLRA_GEMM": "2"})
    out_sk = lin.run(x, dy)
    assert rel_fro(f64(out_sk[0]), f64(out[0])) <= 1e-5
    assert rel_fro(f64(out_sk[3]), f64(out[3])) <= 1e-5


@pytest.mark.parametrize("strategy", [ROW, M.MaterializationStrategy.WeightMaterialize])
def test_cfg5_cb2_layer(strategy):
    """cfg5: the cb2 plugin layer 6656x17920, r=8, 4096 tokens — fused decode in the
    pair kernel (RowMaterialize: Ŵ never in HBM) and the whole-matrix hook path
    (WeightMaterialize) — against the oracle's cb2 decode law."""
    rows, cols, m, r, g = 6656, 17920, 4096, 8, 128
    rng = np.random.default_rng(501)
    codes = rng.integers(0, 1 << 16, (rows, cols // 8), dtype=np.uint32).astype(np.uint16)
    cb = M.default_cb2_codebook()
    scales = (0.01 * (0.5 + rng.random((rows, cols // g)))).astype(np.float32)
    cq = M.Codebook2Quantizer().upload(M.Cb2Matrix(rows, cols, g, codes, cb, scales))
    a32 = (0.02 * rng.standard_normal((rows, r))).astype(np.float32)
    b32 = (0.02 * rng.standard_normal((cols, r))).astype(np.float32)
    layer = M.ModuLoraLayer("cb2", cq, M.LoraAdapter(torch.from_numpy(a32).cuda(),
                                                     torch.from_numpy(b32).cuda(), r, 16.0),
                            strategy=strategy)
    x = _act(60, m, cols)
    dy = _act(61, m, rows)
    y, xb = M.layer_forward(layer, x, out_dtype=torch.float32)
    dx = M.layer_backward(layer, x, xb, dy, dx_dtype=torch.float32)
    da, db = M.grads_of_adapter(layer)

    def deq(xr, gr, chunk=1024):
        yb = np.zeros((xr.shape[0], rows))
        ye = np.zeros_like(yb)
        dxb = np.zeros((gr.shape[0], cols))
        dxe = np.zeros_like(dxb)
        for r0 in range(0, rows, chunk):
            r1 = min(rows, r0 + chunk)
            w32 = orc.cb2_dequantize_f32(codes[r0:r1], r1 - r0, cols, g, cb, scales[r0:r1])
            wex, wbf = w32.astype(np.float64), orc.bf16_round(w32)
            yb[:, r0:r1], ye[:, r0:r1] = xr @ wbf.T, xr @ wex.T
            dxb += gr[:, r0:r1] @ wbf
            dxe += gr[:, r0:r1] @ wex
        return yb, ye, dxb, dxe

    check_layer_pass(deq, a32, b32, 16.0, f64(x), f64(dy), y, xb, dx, da, db,
                     what=f"cfg5 cb2 {M.strategy_name(strategy)}")


def test_cfg1_single_layer_all_kernels(monkeypatch):
    """cfg1 (4096², 4-bit, r=8, m=512) under the cost-model choice, the forced
    1-CTA kernel (256- and 128-token tiles) and the forced pair kernel with stream-K
    and with split-K (distributed fix-up)."""
    lin = Lin(4096, 4096, 4, 8, seed=500, bias=True)
    x = _act(70, 512, 4096)
    dy = _act(71, 512, 4096)
    for env in ({}, {"MLRA_GEMM": "1"}, {"MLRA_GEMM": "3"}, {"MLRA_GEMM": "2", "MLRA_SK": "1"},
                {"MLRA_GEMM": "2", "MLRA_SK": "4"}, {"MLRA_GEMM": "2", "MLRA_SK": "5"}):
        _setenv(monkeypatch, env)
        lin.check(x, dy, lin.run(x, dy), f"cfg1 {env}")
