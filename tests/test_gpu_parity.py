"""GPU parity: the CUDA path (through the C ABI) against the oracle.

Bars:
  * materialize: bit-exact vs (float) of the reference f64 dequantize, and
    bf16 = RN of that (the golden fixtures are the reference's own output);
  * Y / dX tight: normwise rel-Frobenius <= 1e-5 (base GEMM) / 1e-4 (with the
    bf16 LoRA extra-K block) vs an f64 oracle on the same bf16 operands;
  * Y / dX loose: <= 4e-3 vs the exact f64 layer on the same inputs;
  * dA / dB: <= 1e-4 vs the f64 oracle (fp32 intermediates).
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2309_16119_b200 import MlraError
from paper_2309_16119_b200 import modulora as M
from tests.conftest import load_golden, rel_fro
from tests.gpu_util import deq_bf16_f64, f64, qmatrix, random_quantized, to_bf16_dev

pytestmark = pytest.mark.gpu

STRATS = [M.MaterializationStrategy.WeightMaterialize, M.MaterializationStrategy.RowMaterialize,
          M.MaterializationStrategy.QuantizerMatvec]


def _golden_q(gq, i):
    rows, cols, bits, g = (int(v) for v in gq[f"q{i}_meta"])
    return rows, cols, bits, g, gq[f"q{i}_words"], gq[f"q{i}_scales"], gq[f"q{i}_zeros"]


def test_device_is_b200():
    assert M.lib().mlra_device_check() == 0, M.lib().mlra_last_error()


def test_materialize_golden_bit_exact():
    gq = load_golden("quantize.npz")
    i = 0
    while f"q{i}_meta" in gq:
        rows, cols, bits, g, words, sc, z = _golden_q(gq, i)
        dq = M.DeviceQuantizedMatrix(qmatrix(words, rows, cols, bits, g, sc, z))
        want32 = gq[f"q{i}_deq"].astype(np.float32)
        got32 = M.dequantize(dq, torch.float32).cpu().numpy()
        assert np.array_equal(got32.view(np.uint32), want32.view(np.uint32)), f"case {i}"
        got16 = M.dequantize(dq, torch.bfloat16).view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(got16, orc.f32_to_bf16_bits(want32)), f"case {i}"
        # row-wise path (dequantize_row_into)
        r = rows - 1
        assert np.array_equal(M.dequantize_row(dq, r).cpu().numpy(), want32[r])
        with pytest.raises(MlraError) as e:
            M.dequantize_row(dq, rows)
        assert e.value.kind == "RangeError"
        i += 1
    assert i >= 10


@pytest.mark.parametrize("rows,cols,bits", [(4096, 4096, 4), (11008, 4096, 3), (4096, 11008, 3),
                                            (512, 4096, 2), (512, 4096, 8), (256, 17920, 2)])
def test_materialize_llama_shapes_bit_exact(rows, cols, bits):
    q, words, sc, z = random_quantized(rows, cols, bits, 128, seed=rows + cols + bits)
    dq = M.DeviceQuantizedMatrix(q)
    want = orc.dequantize_f32(words, rows, cols, bits, 128, sc, z)
    got = M.dequantize(dq, torch.float32).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    got16 = M.dequantize(dq, torch.bfloat16).view(torch.int16).cpu().numpy().view(np.uint16)
    assert np.array_equal(got16, orc.f32_to_bf16_bits(want))


def test_materialize_pathological_grids_take_exact_f64_path():
    # near-zero group minima: fmaf != (float)f64 for some codes,
    # so these groups must go through the f64 path to stay bit-exact.
    rows, cols, bits, g = 256, 512, 4, 128
    rng = np.random.default_rng(5)
    codes = rng.integers(0, 16, size=rows * cols, dtype=np.uint32)
    words = orc.pack(codes, bits)
    ng = rows * cols // g
    scales = (2.0 ** -7 * (1 + rng.random(ng))).astype(np.float32)
    zeros = (np.sign(rng.random(ng) - 0.5) * 2.0 ** -rng.uniform(20, 60, ng)).astype(np.float32)
    dq = M.DeviceQuantizedMatrix(qmatrix(words, rows, cols, bits, g, scales, zeros))
    assert dq.info()["uncertified_groups"] > 0
    want = orc.dequantize_f32(words, rows, cols, bits, g, scales, zeros)
    got = M.dequantize(dq, torch.float32).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def _lp_check(rows, cols, bits, group, m, strategy, seed):
    q, words, sc, z = random_quantized(rows, cols, bits, group, seed)
    g = cols if group == 0 else group
    dq = M.DeviceQuantizedMatrix(q)
    ctx = M.LpLinearContext(dq, strategy)
    x64 = orc.bf16_round(orc.gaussian(seed + 1, m, cols))
    gy64 = orc.bf16_round(orc.gaussian(seed + 2, m, rows))
    y = f64(M.lp_forward(ctx, to_bf16_dev(x64), out_dtype=torch.float32))
    dx = f64(M.lp_backward(ctx, to_bf16_dev(gy64), out_dtype=torch.float32))
    wbf = deq_bf16_f64(words, rows, cols, bits, g, sc, z)
    assert rel_fro(y, x64 @ wbf.T) <= 1e-5
    assert rel_fro(dx, gy64 @ wbf) <= 1e-5
    wex = orc.dequantize(words, rows, cols, bits, g, sc, z)
    assert rel_fro(y, x64 @ wex.T) <= 4e-3
    assert rel_fro(dx, gy64 @ wex) <= 4e-3
    return y, dx


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("bits", [2, 3, 4, 8])
def test_lp_forward_backward_tiles(bits, strategy):
    _lp_check(256, 512, bits, 128, 300, strategy, seed=40 + bits)


def test_strategies_bit_identical():
    ys = [_lp_check(384, 768, 3, 128, 513, s, seed=77) for s in STRATS]
    for y, dx in ys[1:]:
        assert np.array_equal(y, ys[0][0]) and np.array_equal(dx, ys[0][1])


@pytest.mark.parametrize("rows,cols,bits,group,m", [
    (7, 9, 3, 3, 4), (24, 40, 2, 8, 5), (96, 256, 3, 128, 20), (300, 200, 4, 0, 33),
    (4096, 4096, 4, 128, 512)])
def test_lp_ragged_and_cfg1(rows, cols, bits, group, m):
    _lp_check(rows, cols, bits, group, m, M.MaterializationStrategy.RowMaterialize,
              seed=rows + cols)


def _layer_run(golden, p, strategy, need_dx=True):
    d_out, d_in, bits, g, r, m, has_bias, _ = (int(v) for v in golden[p + "meta"])
    alpha = float(golden[p + "alpha"][0])
    q = qmatrix(golden[p + "words"], d_out, d_in, bits, g, golden[p + "scales"],
                golden[p + "zeros"])
    dq = M.DeviceQuantizedMatrix(q)
    a32 = golden[p + "a"].astype(np.float32)
    b32 = golden[p + "b"].astype(np.float32)
    bias32 = golden[p + "bias"].astype(np.float32) if has_bias else None
    ad = M.LoraAdapter(a=torch.from_numpy(a32).cuda(), b=torch.from_numpy(b32).cuda(), rank=r,
                       alpha=alpha)
    layer = M.ModuLoraLayer("g", dq, ad,
                            bias=None if bias32 is None else torch.from_numpy(bias32).cuda(),
                            bias_trainable=bool(has_bias), strategy=strategy)
    x64 = orc.bf16_round(golden[p + "x"])
    g64 = orc.bf16_round(golden[p + "g"])
    x = to_bf16_dev(x64)
    y, xb = M.layer_forward(layer, x, out_dtype=torch.float32)
    dx = M.layer_backward(layer, x, xb, to_bf16_dev(g64), need_dx=need_dx,
                          dx_dtype=torch.float32)
    w = orc.dequantize(golden[p + "words"], d_out, d_in, bits, g, golden[p + "scales"],
                       golden[p + "zeros"])
    # exact f64 reference layer on the same (bf16 activations, fp32 adapter) inputs
    yr, xbr = orc.layer_forward(w, a32, b32, alpha, bias32, x64)
    dxr, dar, dbr, dbiasr = orc.layer_backward(w, a32, b32, alpha, x64, xbr, g64, need_dx=need_dx,
                                               need_dbias=bool(has_bias))
    return dict(layer=layer, y=f64(y), xb=f64(xb), dx=None if dx is None else f64(dx),
                yr=yr, xbr=xbr, dxr=dxr, dar=dar, dbr=dbr, dbiasr=dbiasr)


@pytest.mark.parametrize("strategy", STRATS)
def test_layer_golden_cases(strategy):
    gl = load_golden("layer.npz")
    i = 0
    while f"l{i}_meta" in gl:
        p = f"l{i}_"
        need_dx = bool(gl[p + "meta"][7])
        o = _layer_run(gl, p, strategy, need_dx)
        assert rel_fro(o["xb"], o["xbr"]) <= 1e-5, i
        assert rel_fro(o["y"], o["yr"]) <= 4e-3, i
        if need_dx:
            assert rel_fro(o["dx"], o["dxr"]) <= 4e-3, i
        else:
            assert o["dx"] is None
        da, db = M.grads_of_adapter(o["layer"])
        assert rel_fro(f64(da), o["dar"]) <= 1e-4, i
        assert rel_fro(f64(db), o["dbr"]) <= 1e-4, i
        if o["dbiasr"] is not None:
            assert rel_fro(f64(o["layer"].grad_bias), o["dbiasr"]) <= 1e-5, i
        i += 1
    assert i == 6


@pytest.mark.parametrize("d_out,d_in,bits,r,m", [(4096, 4096, 4, 8, 512), (1024, 2816, 3, 16, 700),
                                                 (512, 1024, 4, 64, 256), (256, 512, 2, 100, 64)])
def test_layer_llama_shapes(d_out, d_in, bits, r, m):
    seed = d_out + d_in + r
    q, words, sc, z = random_quantized(d_out, d_in, bits, 128, seed)
    dq = M.DeviceQuantizedMatrix(q)
    alpha = 32.0
    s = alpha / r
    a32 = orc.gaussian(seed + 1, d_out, r, 0.0, 0.02).astype(np.float32)
    b32 = orc.gaussian(seed + 2, d_in, r, 0.0, 0.02).astype(np.float32)
    ad = M.LoraAdapter(a=torch.from_numpy(a32).cuda(), b=torch.from_numpy(b32).cuda(), rank=r,
                       alpha=alpha)
    layer = M.ModuLoraLayer("l", dq, ad, strategy=M.MaterializationStrategy.RowMaterialize)
    x64 = orc.bf16_round(orc.gaussian(seed + 3, m, d_in))
    g64 = orc.bf16_round(orc.gaussian(seed + 4, m, d_out))
    x = to_bf16_dev(x64)
    y, xb = M.layer_forward(layer, x, out_dtype=torch.float32)
    dx = M.layer_backward(layer, x, xb, to_bf16_dev(g64), dx_dtype=torch.float32)
    wbf = deq_bf16_f64(words, d_out, d_in, bits, 128, sc, z)
    A, B = a32.astype(np.float64), b32.astype(np.float64)
    xbr = x64 @ B
    dyar = g64 @ A
    # tight: the GPU recipe (bf16 Ŵ, bf16(s·xb), bf16 A / B) in f64
    y_recipe = x64 @ wbf.T + orc.bf16_round(s * xbr) @ orc.bf16_round(A).T
    dx_recipe = g64 @ wbf + orc.bf16_round(s * dyar) @ orc.bf16_round(B).T
    assert rel_fro(f64(xb), xbr) <= 1e-5
    assert rel_fro(f64(y), y_recipe) <= 1e-4
    assert rel_fro(f64(dx), dx_recipe) <= 1e-4
    # loose: exact f64 layer (sampled rows for the O(m·N·K) part)
    wex = orc.dequantize(words, d_out, d_in, bits, 128, sc, z)
    rows = np.arange(0, m, max(1, m // 16))
    assert rel_fro(f64(y)[rows], x64[rows] @ wex.T + s * xbr[rows] @ A.T) <= 4e-3
    assert rel_fro(f64(dx)[rows], g64[rows] @ wex + s * dyar[rows] @ B.T) <= 4e-3
    da, db = M.grads_of_adapter(layer)
    assert rel_fro(f64(da), s * g64.T @ xbr) <= 1e-4
    assert rel_fro(f64(db), s * x64.T @ dyar) <= 1e-4


def test_bf16_outputs_and_autograd_function():
    d_out, d_in, r, m = 512, 768, 16, 333
    q, words, sc, z = random_quantized(d_out, d_in, 4, 128, 3)
    dq = M.DeviceQuantizedMatrix(q)
    a = (torch.randn(d_out, r) * 0.02).cuda()
    b = (torch.randn(d_in, r) * 0.02).cuda()
    layer = M.ModuLoraLayer("f", dq, M.LoraAdapter(a=a, b=b, rank=r, alpha=16.0))
    x = torch.randn(m, d_in).to(torch.bfloat16).cuda().requires_grad_(True)
    y = M.ModuLoraLinearFunction.apply(x, a, b, None, layer)
    assert y.dtype == torch.bfloat16 and y.shape == (m, d_out)
    y.float().sum().backward()
    assert x.grad is not None and x.grad.shape == x.shape
    wbf = torch.from_numpy(deq_bf16_f64(words, d_out, d_in, 4, 128, sc, z)).cuda()
    ones = torch.ones(m, d_out, dtype=torch.float64, device="cuda")
    want_dx = ones @ wbf + ((16.0 / r) * ones @ a.double()) @ b.double().T
    assert rel_fro(f64(x.grad), want_dx.cpu().numpy()) <= 8e-3


def test_empty_tokens_and_errors():
    q, *_ = random_quantized(256, 256, 4, 128, 9)
    dq = M.DeviceQuantizedMatrix(q)
    ctx = M.LpLinearContext(dq, M.MaterializationStrategy.RowMaterialize)
    y = M.lp_forward(ctx, torch.empty(0, 256, dtype=torch.bfloat16, device="cuda"))
    assert y.shape == (0, 256)
    with pytest.raises(MlraError) as e:
        M.lp_forward(ctx, torch.zeros(4, 255, dtype=torch.bfloat16, device="cuda"))
    assert e.value.kind == "DimensionError"
    with pytest.raises(MlraError) as e:
        M.lp_forward(M.LpLinearContext(None), torch.zeros(4, 256, dtype=torch.bfloat16, device="cuda"))
    assert e.value.kind == "ContractError"
    layer = M.make_layer("e", dq, 4, 8.0, 1)
    with pytest.raises(MlraError) as e:
        M.grads_of_adapter(layer)
    assert e.value.kind == "ContractError"
    # a fresh layer (A = 0) computes exactly the frozen base (test_lora.cpp:91-105)
    x = torch.randn(40, 256).to(torch.bfloat16).cuda()
    y1, _ = M.layer_forward(layer, x, out_dtype=torch.float32)
    y0 = M.lp_forward(ctx, x, out_dtype=torch.float32)
    assert torch.equal(y1, y0)


@pytest.mark.parametrize("bits,mn", [(3, False), (3, True), (4, False), (2, True)])
def test_pair_kernel_matches_single_cta(bits, mn, monkeypatch):
    """The CTA-pair (cta_group::2) GEMM and the 1-CTA GEMM compute the same
    products on the same bf16 operands (same K order) -> identical outputs."""
    rows, cols, m = 768, 1024, 1100
    q, words, sc, z = random_quantized(rows, cols, bits, 128, seed=bits + 10 * mn)
    dq = M.DeviceQuantizedMatrix(q)
    ctx = M.LpLinearContext(dq, M.MaterializationStrategy.RowMaterialize)
    a = to_bf16_dev(orc.bf16_round(orc.gaussian(5, m, rows if mn else cols)))
    outs = []
    monkeypatch.setenv("MLRA_SK", "0")  # whole tiles: same K order as the 1-CTA kernel
    for mode in ("1", "2", "3"):
        monkeypatch.setenv("MLRA_GEMM", mode)
        f = M.lp_backward if mn else M.lp_forward
        outs.append(f64(f(ctx, a, out_dtype=torch.float32)))
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    wbf = deq_bf16_f64(words, rows, cols, bits, 128, sc, z)
    ref = f64(a) @ (wbf if mn else wbf.T)
    assert rel_fro(outs[1], ref) <= 1e-5


@pytest.mark.parametrize("rows,cols,m,bits,mn", [
    (768, 1024, 1100, 3, False),   # 9 tiles x 16 k-blocks over 18 pairs: 2-3 pairs per tile
    (768, 1024, 1100, 4, True),
    (4096, 4096, 1024, 3, False),  # 32 tiles over 74 pairs
    (4096, 4096, 1024, 4, True),
    (512, 4096, 512, 2, False),    # 2 tiles x 64 k-blocks: one tile cut among ~8 pairs
])
def test_stream_k_matches_whole_tiles(rows, cols, m, bits, mn, monkeypatch):
    """Stream-K (tile x k-block ranges per CTA pair, split tiles finished from
    fp32 partials) computes the same products as the whole-tile schedule; only
    the fp32 summation order across the cut differs."""
    q, words, sc, z = random_quantized(rows, cols, bits, 128, seed=rows + m + bits + 7 * mn)
    dq = M.DeviceQuantizedMatrix(q)
    ctx = M.LpLinearContext(dq, M.MaterializationStrategy.RowMaterialize)
    a = to_bf16_dev(orc.bf16_round(orc.gaussian(9, m, rows if mn else cols)))
    f = M.lp_backward if mn else M.lp_forward
    monkeypatch.setenv("MLRA_GEMM", "2")
    outs = {}
    # whole tiles, stream-K, split-K on 512- and on 256-token tiles (all-warp fix-up)
    for sk in ("0", "1", "4", "5"):
        monkeypatch.setenv("MLRA_SK", sk)
        outs[sk] = f64(f(ctx, a, out_dtype=torch.float32))
    for sk in ("1", "4", "5"):
        assert rel_fro(outs[sk], outs["0"]) <= 1e-5  # fp32 order across the cut (~sqrt(K) ulp)
    for sk in ("4", "5"):  # the split fix-up adds partials in pair order: repeatable
        monkeypatch.setenv("MLRA_SK", sk)
        assert np.array_equal(f64(f(ctx, a, out_dtype=torch.float32)), outs[sk])
    wbf = deq_bf16_f64(words, rows, cols, bits, 128, sc, z)
    ref = f64(a) @ (wbf if mn else wbf.T)
    assert rel_fro(outs["1"], ref) <= 1e-5
    # repeatable: the owner adds partials in pair order
    monkeypatch.setenv("MLRA_SK", "1")
    assert np.array_equal(f64(f(ctx, a, out_dtype=torch.float32)), outs["1"])
    # the all-warp owner fix-up and the 4-epilogue-warp one sum in the same order
    monkeypatch.setenv("MLRA_SK_OWNER4", "1")
    assert np.array_equal(f64(f(ctx, a, out_dtype=torch.float32)), outs["1"])
    y4 = f64(f(ctx, a))  # bf16 output (paired-row stores)
    monkeypatch.delenv("MLRA_SK_OWNER4")
    assert np.array_equal(f64(f(ctx, a)), y4)


def test_stream_k_layer_with_lora_and_bias(monkeypatch):
    """Split tiles whose cut falls next to the LoRA k-block, with bias."""
    d_out, d_in, r, m, bits = 1024, 1536, 24, 900, 3
    q, words, sc, z = random_quantized(d_out, d_in, bits, 128, seed=77)
    dq = M.DeviceQuantizedMatrix(q)
    a32 = orc.gaussian(78, d_out, r, 0.0, 0.02).astype(np.float32)
    b32 = orc.gaussian(79, d_in, r, 0.0, 0.02).astype(np.float32)
    bias = orc.gaussian(80, 1, d_out).astype(np.float32)[0]
    x = to_bf16_dev(orc.bf16_round(orc.gaussian(81, m, d_in)))
    g = to_bf16_dev(orc.bf16_round(orc.gaussian(82, m, d_out)))
    monkeypatch.setenv("MLRA_GEMM", "2")
    res = {}
    for sk in ("0", "1", "4", "5", "1o4"):
        monkeypatch.setenv("MLRA_SK", sk[0])
        monkeypatch.setenv("MLRA_SK_OWNER4", "1" if sk == "1o4" else "0")
        ad = M.LoraAdapter(a=torch.from_numpy(a32).cuda(), b=torch.from_numpy(b32).cuda(), rank=r,
                           alpha=32.0)
        layer = M.ModuLoraLayer("k", dq, ad, bias=torch.from_numpy(bias).cuda(),
                                strategy=M.MaterializationStrategy.RowMaterialize)
        y, xb = M.layer_forward(layer, x, out_dtype=torch.float32)
        dx = M.layer_backward(layer, x, xb, g, dx_dtype=torch.float32)
        res[sk] = (f64(y), f64(dx))
    for sk in ("1", "4", "5"):
        assert rel_fro(res[sk][0], res["0"][0]) <= 1e-5
        assert rel_fro(res[sk][1], res["0"][1]) <= 1e-5
    # stream-K owner fix-up: all 16 warps vs the 4 epilogue warps, same bits
    assert np.array_equal(res["1"][0], res["1o4"][0]) and np.array_equal(res["1"][1], res["1o4"][1])


@pytest.mark.parametrize("strategy", STRATS)
def test_identity_and_one_hot_exact(strategy):
    # test_lowprec.cpp:73-96: identity weights pass x and g through exactly; a one-hot
    # input reads out one column of the dequantized weights exactly
    n = 256
    codes = np.zeros((n, n), np.uint32)
    codes[np.arange(n), np.arange(n)] = 1
    words = orc.pack(codes.ravel(), 8)
    dq = M.DeviceQuantizedMatrix(qmatrix(words, n, n, 8, n, np.ones(n, np.float32),
                                         np.zeros(n, np.float32)))
    ctx = M.LpLinearContext(dq, strategy)
    x64 = orc.bf16_round(orc.gaussian(3, 40, n))
    x = to_bf16_dev(x64)
    assert np.array_equal(f64(M.lp_forward(ctx, x, torch.float32)), x64)
    assert np.array_equal(f64(M.lp_backward(ctx, x, torch.float32)), x64)
    q, words, sc, z = random_quantized(384, 512, 3, 128, seed=12)
    dq = M.DeviceQuantizedMatrix(q)
    wb = deq_bf16_f64(words, 384, 512, 3, 128, sc, z)
    k = 137
    e = np.zeros((3, 512))
    e[:, k] = 1.0
    y = f64(M.lp_forward(M.LpLinearContext(dq, strategy), to_bf16_dev(e), torch.float32))
    assert np.array_equal(y[0], wb[:, k])


def test_fresh_adapter_equals_base_and_zero_base():
    # test_lora.cpp:91-150: with A = 0 (the init) the layer is the base linear; a
    # zero base leaves only the adapter term
    d_out, d_in, r, m = 512, 768, 8, 100
    q, words, sc, z = random_quantized(d_out, d_in, 4, 128, seed=21)
    dq = M.DeviceQuantizedMatrix(q)
    layer = M.make_layer("fresh", dq, r, 16.0, seed=3)
    x = to_bf16_dev(orc.bf16_round(orc.gaussian(22, m, d_in)))
    y, _ = M.layer_forward(layer, x, out_dtype=torch.float32)
    base = M.lp_forward(M.LpLinearContext(dq, M.MaterializationStrategy.RowMaterialize), x,
                        torch.float32)
    assert torch.equal(y, base)
    zq = qmatrix(orc.pack(np.zeros(d_out * d_in, np.uint32), 2), d_out, d_in, 2, 128,
                 np.ones(d_out * d_in // 128, np.float32), np.zeros(d_out * d_in // 128, np.float32))
    zl = M.ModuLoraLayer("zero", M.DeviceQuantizedMatrix(zq),
                         M.LoraAdapter((torch.randn(d_out, r) * 0.1).cuda(),
                                       (torch.randn(d_in, r) * 0.1).cuda(), r, 16.0))
    yz, xb = M.layer_forward(zl, x, out_dtype=torch.float32)
    s = 16.0 / r
    ref = orc.bf16_round(s * f64(xb)) @ orc.bf16_round(f64(zl.adapter.a)).T
    assert rel_fro(f64(yz), ref) <= 1e-5


@pytest.mark.parametrize("d_out,d_in,r,m,bias", [(1024, 2816, 16, 700, True), (4096, 4096, 8, 512, False),
                                                 (512, 1024, 100, 4100, True), (256, 512, 8, 1, True)])
def test_adapter_gradients_bitwise_reproducible(d_out, d_in, r, m, bias):
    """the skinny products reduce in a fixed order (no atomics), so
    xb, dA, dB, dbias, Y and dX are bitwise equal run to run, as the reference's
    fixed-order loops are (matrix.cpp:81-97; test_train.cpp:328-387 asserts
    bit-equal training trajectories)."""
    q, *_ = random_quantized(d_out, d_in, 3, 128, seed=d_out + r)
    dq = M.DeviceQuantizedMatrix(q)
    a = (torch.randn(d_out, r, generator=torch.Generator().manual_seed(1)) * 0.02).cuda()
    b = (torch.randn(d_in, r, generator=torch.Generator().manual_seed(2)) * 0.02).cuda()
    layer = M.ModuLoraLayer("det", dq, M.LoraAdapter(a, b, r, 16.0),
                            bias=torch.zeros(d_out).cuda() if bias else None, bias_trainable=bias)
    x = torch.randn(m, d_in, generator=torch.Generator().manual_seed(3)).to(torch.bfloat16).cuda()
    dy = torch.randn(m, d_out, generator=torch.Generator().manual_seed(4)).to(torch.bfloat16).cuda()
    runs = []
    for _ in range(3):
        y, xb = M.layer_forward(layer, x)
        dx = M.layer_backward(layer, x, xb, dy)
        da, db = (t.clone() for t in M.grads_of_adapter(layer))
        runs.append((y, xb, dx, da, db, None if layer.grad_bias is None else layer.grad_bias.clone()))
        torch.cuda.synchronize()
    for other in runs[1:]:
        for u, v in zip(runs[0], other):
            assert (u is None and v is None) or torch.equal(u, v)


@pytest.mark.parametrize("d_out,d_in,r,m", [
    (1024, 1024, 16, 4100),  # ragged last token tile
    (512, 384, 8, 300),      # 6 reduction chunks over 8 CTAs: empty ranges
    (768, 4096, 64, 2048),   # NT = 8 (fused only when forced: MLRA_THIN_CL=1)
    (768, 4096, 72, 2048),   # r = 72: the range kernel under both settings
    (256, 512, 8, 1),
])
def test_row_products_cluster_vs_range_kernel(d_out, d_in, r, m, monkeypatch):
    """The row products (xb = x·B, dyA = dy·A and their derived GEMM operands /
    transposed planes) on the cluster kernel (k_rowmma_cl: kThinCl CTAs split one
    token tile's reduction, DSMEM reduction in rank order) and on the range
    kernel: both match the f64 oracle to fp32-order rounding, and each is bitwise
    repeatable."""
    q, words, sc, z = random_quantized(d_out, d_in, 3, 128, seed=d_out + d_in + r)
    dq = M.DeviceQuantizedMatrix(q)
    a = (torch.randn(d_out, r, generator=torch.Generator().manual_seed(5)) * 0.02).cuda()
    b = (torch.randn(d_in, r, generator=torch.Generator().manual_seed(6)) * 0.02).cuda()
    layer = M.ModuLoraLayer("cl", dq, M.LoraAdapter(a, b, r, 16.0))
    x = to_bf16_dev(orc.bf16_round(orc.gaussian(7, m, d_in)))
    dy = to_bf16_dev(orc.bf16_round(orc.gaussian(8, m, d_out)))
    res = {}
    for cl in ("0", "1"):
        monkeypatch.setenv("MLRA_THIN_CL", cl)
        outs = []
        for _ in range(2):
            y, xb = M.layer_forward(layer, x, out_dtype=torch.float32)
            dx = M.layer_backward(layer, x, xb, dy, dx_dtype=torch.float32)
            outs.append([f64(t) for t in (y, xb, dx, *M.grads_of_adapter(layer))])
        for u, v in zip(*outs):
            assert np.array_equal(u, v)
        res[cl] = outs[0]
    s = 16.0 / r
    xb_ref = f64(x) @ f64(b)
    dya_ref = f64(dy) @ f64(a)
    wbf = deq_bf16_f64(words, d_out, d_in, 3, 128, sc, z)
    y_ref = f64(x) @ wbf.T + orc.bf16_round(s * xb_ref) @ orc.bf16_round(f64(a)).T
    dx_ref = f64(dy) @ wbf + orc.bf16_round(s * dya_ref) @ orc.bf16_round(f64(b)).T
    db_ref = s * f64(x).T @ dya_ref
    for cl in ("0", "1"):
        y, xb, dx, da, db = res[cl]
        assert rel_fro(xb, xb_ref) <= 1e-5, cl
        assert rel_fro(db, db_ref) <= 1e-5, cl
        # bf16(s·xb) / bf16(s·dyA) may round differently from the f64 reference's
        assert rel_fro(y, y_ref) <= 1e-3 and rel_fro(dx, dx_ref) <= 1e-3, cl
    for u, v in zip(res["0"], res["1"]):  # fp32 summation order only
        assert rel_fro(u, v) <= 1e-3


def test_workspace_arena_across_streams_sizes_and_capture():
    """The per-stream workspace arena (capi.cu Scratch): a pass gives the same bits
    on any stream, across arena regrowth (small -> large -> small on one stream),
    and under CUDA graph capture (which takes the pool path)."""

    def make(d_out, d_in, r, seed):
        q, *_ = random_quantized(d_out, d_in, 3, 128, seed=seed)
        a = (torch.randn(d_out, r, generator=torch.Generator().manual_seed(seed)) * 0.02).cuda()
        b = (torch.randn(d_in, r, generator=torch.Generator().manual_seed(seed + 1)) * 0.02).cuda()
        return M.ModuLoraLayer("arena", M.DeviceQuantizedMatrix(q), M.LoraAdapter(a, b, r, 16.0))

    def run(layer, m, seed):
        x = torch.randn(m, layer.d_in(), generator=torch.Generator().manual_seed(seed)).to(torch.bfloat16).cuda()
        dy = torch.randn(m, layer.d_out(), generator=torch.Generator().manual_seed(seed + 7)).to(torch.bfloat16).cuda()
        y, xb = M.layer_forward(layer, x)
        dx = M.layer_backward(layer, x, xb, dy)
        return [t.clone() for t in (y, xb, dx, *M.grads_of_adapter(layer))]

    small, big = make(256, 512, 8, 11), make(4096, 4096, 16, 12)
    ref_small, ref_big = run(small, 300, 1), run(big, 1024, 2)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for st, layer, m, seed, ref in ((s1, small, 300, 1, ref_small), (s2, big, 1024, 2, ref_big),
                                    (s1, big, 1024, 2, ref_big), (s1, small, 300, 1, ref_small)):
        with torch.cuda.stream(st):
            got = run(layer, m, seed)
        st.synchronize()
        for u, v in zip(got, ref):
            assert torch.equal(u, v)
    # graph capture (pool path), replayed
    x = torch.randn(300, 512, generator=torch.Generator().manual_seed(1)).to(torch.bfloat16).cuda()
    M.layer_forward(small, x)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        yg, xbg = M.layer_forward(small, x)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(yg, ref_small[0]) and torch.equal(xbg, ref_small[1])


@pytest.mark.parametrize("env", [{"MLRA_PDL": "0"}, {"MLRA_DA_EARLY": "0"}, {"MLRA_SIDE_FIRST": "1"},
                                 {"MLRA_NO_SIDE": "1"}, {"MLRA_THIN_MAXC": "1000"},
                                 {"MLRA_THIN_CL": "1"}])
def test_launch_switches_bit_identical(env, tmp_path):
    """The launch-order / launch-mode switches (programmatic dependent launch, the
    side-stream schedule of dA/dB, the skinny-product CTA cap) change only when
    kernels run, never what they compute: bitwise-equal outputs."""
    import os
    import subprocess
    import sys
    helper = os.path.join(os.path.dirname(__file__), "helpers", "layer_pass_dump.py")
    ref_p, alt_p = tmp_path / "ref.npz", tmp_path / "alt.npz"
    base = {k: v for k, v in os.environ.items() if not k.startswith("MLRA_")}
    for path, extra in ((ref_p, {}), (alt_p, env)):
        r = subprocess.run([sys.executable, helper, str(path)], env=dict(base, **extra),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
    ref, alt = np.load(ref_p), np.load(alt_p)
    for k in ref.files:
        if env.get("MLRA_THIN_MAXC") or env.get("MLRA_THIN_CL"):
            # a different CTA count (or the cluster row-product kernel) changes the skinny products' fp32 summation order (and
            # through bf16(s·xb) the bf16 outputs by at most an ulp here and there)
            bound = 1e-3 if k.split("_")[0] in ("y", "dx") else 1e-5
            assert rel_fro(alt[k].astype(np.float64), ref[k].astype(np.float64)) <= bound, k
        else:
            assert np.array_equal(ref[k], alt[k]), k
