"""The device Quantizer plugin: the black-box dequant hook and
the built-in non-affine "cb2" codebook plugin.

CPU tests pin the cb2 decode law (oracle/mlra_oracle.c orc_cb2_dequant_f32)
with hand-computed known answers and a pure-Python restatement; GPU tests
check the library's cb2 materialize kernel bit-exactly against that oracle,
the hook-driven GEMMs (slabbed materialization through the hook + tcgen05)
against an f64 oracle on the same bf16 operands, and re-express the
reference's hook dispatch test (DoublingQuantizer, test_lowprec.cpp:354-377).
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2309_16119_b200 import MlraError
from paper_2309_16119_b200 import modulora as M
from tests.conftest import rel_fro
from tests.gpu_util import f64, random_quantized, to_bf16_dev

S = M.MaterializationStrategy


def _py_cb2(codes, rows, cols, group, cb, scales):
    out = np.empty((rows, cols), np.float32)
    for i in range(rows):
        for u in range(cols // 8):
            c = int(codes[i, u])
            for j in range(8):
                m = np.float32(cb[c & 0xFF, j])
                if (c >> (8 + j)) & 1:
                    m = -m
                out[i, 8 * u + j] = np.float32(scales[i, (8 * u + j) // group]) * m
    return out


def _random_cb2(rows, cols, group, seed):
    rng = np.random.default_rng(seed)
    codes = rng.integers(0, 1 << 16, size=(rows, cols // 8), dtype=np.uint32).astype(np.uint16)
    cb = M.default_cb2_codebook()
    scales = (0.01 * (0.5 + rng.random((rows, cols // group)))).astype(np.float32)
    return M.Cb2Matrix(rows, cols, group, codes, cb, scales)


# ----------------------------------------------------------------------------- CPU
def test_cb2_known_answer():
    cb = np.zeros((256, 8), np.float32)
    cb[3] = [0.5, 1.5, 2.5, 3.5, 0.25, 0.0, 1.0, 2.0]
    cb[255] = 1.0
    # row 0: code 3, signs on entries 1 and 7; row 1: code 255 all negative, then code 3 no sign
    codes = np.array([[3 | (1 << 9) | (1 << 15), 3], [255 | (0xFF << 8), 3]], np.uint16)
    scales = np.array([[2.0, 0.5], [4.0, 3.0]], np.float32)  # group 8
    got = orc.cb2_dequantize_f32(codes, 2, 16, 8, cb, scales)
    want = np.array([
        [1.0, -3.0, 5.0, 7.0, 0.5, 0.0, 2.0, -4.0, 0.25, 0.75, 1.25, 1.75, 0.125, 0.0, 0.5, 1.0],
        [-4.0] * 8 + [1.5, 4.5, 7.5, 10.5, 0.75, 0.0, 3.0, 6.0]], np.float32)
    assert np.array_equal(got, want)


def test_cb2_oracle_matches_python_restatement():
    m = _random_cb2(6, 48, 16, seed=3)
    got = orc.cb2_dequantize_f32(m.codes, 6, 48, 16, m.codebook, m.scales)
    want = _py_cb2(m.codes, 6, 48, 16, m.codebook, m.scales)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_default_codebook_is_a_sorted_shell():
    cb = M.default_cb2_codebook()
    assert cb.shape == (256, 8) and cb.dtype == np.float32
    assert len({tuple(r) for r in cb}) == 256
    n = (cb.astype(np.float64) ** 2).sum(1)
    assert np.all(np.diff(n) >= 0) and np.all(cb > 0)


def test_cb2_quantizer_roundtrip_error():
    w = orc.gaussian(7, 32, 256, 0.0, 0.02)
    qz = M.Codebook2Quantizer()
    assert qz.name() == "cb2"
    m = qz.quantize(w, None, 2, 128)
    assert m.codes.shape == (32, 32) and m.scales.shape == (32, 2)
    d = orc.cb2_dequantize_f32(m.codes, 32, 256, 128, m.codebook, m.scales)
    assert rel_fro(d, w) < 0.36  # 2 bits / weight on Gaussian groups
    with pytest.raises(MlraError) as e:
        qz.quantize(w, None, 3, 128)
    assert e.value.kind == "ConfigError"


# ----------------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,group", [(6656, 17920, 128), (300, 1000, 40), (7, 64, 64)])
def test_cb2_materialize_bit_exact(rows, cols, group):
    m = _random_cb2(rows, cols, group, seed=rows)
    dq = M.Codebook2Quantizer().upload(m)
    want = orc.cb2_dequantize_f32(m.codes, rows, cols, group, m.codebook, m.scales)
    got = M.dequantize(dq, torch.float32).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    got16 = M.dequantize(dq, torch.bfloat16).view(torch.int16).cpu().numpy().view(np.uint16)
    assert np.array_equal(got16, orc.f32_to_bf16_bits(want))
    # tiles (the hook's unit of work), including an unaligned leading dimension
    r0, c0 = rows // 3, (cols // 3) // 8 * 8
    nr, nc = rows - r0, (cols - c0) // 16 * 8
    out = torch.zeros(nr, nc + 3, dtype=torch.float32, device="cuda")
    M.dequantize_tile(dq, r0, nr, c0, nc, torch.float32, out=out[:, :nc])
    assert np.array_equal(out[:, :nc].cpu().numpy(), want[r0:, c0:c0 + nc])
    assert not out[:, nc:].any()


@pytest.mark.gpu
def test_cb2_validation_errors():
    m = _random_cb2(16, 64, 32, seed=1)
    bad = M.Cb2Matrix(16, 64, 32, m.codes, m.codebook, -m.scales)
    with pytest.raises(MlraError) as e:
        M.Codebook2Quantizer().upload(bad)
    assert e.value.kind == "NumericError"
    with pytest.raises(MlraError) as e:
        M.Codebook2Quantizer().upload(M.Cb2Matrix(16, 64, 12, m.codes, m.codebook, m.scales[:, :1]))
    assert e.value.kind in ("ConfigError", "FormatError")
    dq = M.Codebook2Quantizer().upload(m)
    with pytest.raises(MlraError) as e:
        M.dequantize_tile(dq, 0, 17, 0, 8)
    assert e.value.kind == "RangeError"


def _deq_bf16(dq):
    return f64(M.dequantize(dq, torch.bfloat16))


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", list(S))
@pytest.mark.parametrize("slab_mb", [0, 1])
def test_cb2_lp_forward_backward(strategy, slab_mb, monkeypatch):
    if slab_mb:
        monkeypatch.setenv("MLRA_SLAB_MB", str(slab_mb))  # force several slabs
    d_out, d_in, m = 1280, 768, 300
    w = orc.gaussian(11, d_out, d_in, 0.0, 0.02)
    dq = M.Codebook2Quantizer().upload(M.Codebook2Quantizer().quantize(w, None, 2, 128))
    wb = _deq_bf16(dq)
    x = orc.bf16_round(orc.gaussian(12, m, d_in))
    g = orc.bf16_round(orc.gaussian(13, m, d_out))
    ctx = M.LpLinearContext(dq, strategy)
    y = f64(M.lp_forward(ctx, to_bf16_dev(x), out_dtype=torch.float32))
    dx = f64(M.lp_backward(ctx, to_bf16_dev(g), out_dtype=torch.float32))
    assert rel_fro(y, x @ wb.T) < 1e-5
    assert rel_fro(dx, g @ wb) < 1e-5
    if strategy != S.WeightMaterialize and slab_mb:
        assert ctx.ledger_bytes() < d_out * d_in * 2


@pytest.mark.gpu
def test_cb2_layer_forward_backward():
    d_out, d_in, m, r, alpha = 1024, 2048, 512, 8, 16.0
    w = orc.gaussian(21, d_out, d_in, 0.0, 0.02)
    dq = M.Codebook2Quantizer().upload(M.Codebook2Quantizer().quantize(w, None, 2, 128))
    wb = _deq_bf16(dq)
    a = orc.gaussian(22, d_out, r, 0.0, 0.5).astype(np.float32)
    b = orc.gaussian(23, d_in, r, 0.0, 0.02).astype(np.float32)
    x = orc.bf16_round(orc.gaussian(24, m, d_in))
    g = orc.bf16_round(orc.gaussian(25, m, d_out))
    for strategy in S:
        layer = M.ModuLoraLayer("cb2", dq, M.LoraAdapter(torch.from_numpy(a).cuda(),
                                                          torch.from_numpy(b).cuda(), r, alpha),
                                strategy=strategy)
        y, xb = M.layer_forward(layer, to_bf16_dev(x), out_dtype=torch.float32)
        dx = M.layer_backward(layer, to_bf16_dev(x), xb, to_bf16_dev(g), dx_dtype=torch.float32)
        yr, xbr = orc.layer_forward(wb, a, b, alpha, None, x)
        dxr, dar, dbr, _ = orc.layer_backward(wb, a, b, alpha, x, xbr, g)
        da, db = M.grads_of_adapter(layer)
        s = alpha / r
        A, B = a.astype(np.float64), b.astype(np.float64)
        # tight: the GPU recipe (bf16 Ŵ, bf16(s·xb), bf16 A / B) in f64; loose: exact layer
        y_recipe = x @ wb.T + orc.bf16_round(s * (x @ B)) @ orc.bf16_round(A).T
        dx_recipe = g @ wb + orc.bf16_round(s * (g @ A)) @ orc.bf16_round(B).T
        assert rel_fro(f64(y), y_recipe) < 1e-4 and rel_fro(f64(y), yr) < 4e-3
        assert rel_fro(f64(dx), dx_recipe) < 1e-4 and rel_fro(f64(dx), dxr) < 4e-3
        assert rel_fro(f64(da), dar) < 1e-4 and rel_fro(f64(db), dbr) < 1e-4


@pytest.mark.gpu
def test_matvec_hook_dispatch_doubling_quantizer():
    # test_lowprec.cpp:354-377: QuantizerMatvec delegates to the hook (outputs
    # double); WeightMaterialize (and the fused row path) ignore it.
    q, *_ = random_quantized(640, 384, 4, 128, seed=33)
    dq = M.DeviceQuantizedMatrix(q)
    x = to_bf16_dev(orc.bf16_round(orc.gaussian(34, 96, 384)))
    g = to_bf16_dev(orc.bf16_round(orc.gaussian(35, 96, 640)))
    hook = M.DoublingQuantizer()
    plain = M.LpLinearContext(dq, S.QuantizerMatvec)
    hooked = M.LpLinearContext(dq, S.QuantizerMatvec, matvec_hook=hook)
    y0 = M.lp_forward(plain, x, torch.float32)
    y1 = M.lp_forward(hooked, x, torch.float32)
    assert rel_fro(f64(y1), 2 * f64(y0)) < 1e-6
    dx0 = M.lp_backward(plain, g, torch.float32)
    dx1 = M.lp_backward(hooked, g, torch.float32)
    assert rel_fro(f64(dx1), 2 * f64(dx0)) < 1e-6
    for s in (S.WeightMaterialize, S.RowMaterialize):
        yw = M.lp_forward(M.LpLinearContext(dq, s, matvec_hook=hook), x, torch.float32)
        yp = M.lp_forward(M.LpLinearContext(dq, s), x, torch.float32)
        assert torch.equal(yw, yp)


@pytest.mark.gpu
def test_python_plugin_on_opaque_matrix():
    # a user plugin that owns its packed format: here a dense bf16 table
    table = torch.randn(512, 256, device="cuda").to(torch.bfloat16)

    class DenseTable(M.QuantizerHook):
        def materialize(self, q, row0, nrows, col0, ncols, out, stream):
            with torch.cuda.stream(stream):
                out.copy_(table[row0:row0 + nrows, col0:col0 + ncols].to(out.dtype))

    dq = M.DeviceQuantizedMatrix.opaque(512, 256, 16, DenseTable())
    assert torch.equal(M.dequantize(dq, torch.bfloat16), table)
    x = torch.randn(300, 256, device="cuda").to(torch.bfloat16)
    for s in S:
        y = M.lp_forward(M.LpLinearContext(dq, s), x, torch.float32)
        ref = x.double() @ table.double().T
        assert rel_fro(f64(y), ref.cpu().numpy()) < 1e-5

    class Broken(M.QuantizerHook):
        def materialize(self, *a):
            raise RuntimeError("plugin failure")

    bq = M.DeviceQuantizedMatrix.opaque(256, 256, 2, Broken())
    with pytest.raises(MlraError) as e:
        M.lp_forward(M.LpLinearContext(bq, S.RowMaterialize), x[:, :256], torch.float32)
    assert e.value.kind == "ContractError"


# ----------------------------------------------------------------------------- RTN
@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,bits,group", [(7, 9, 3, 0), (7, 9, 3, 3), (64, 96, 2, 32),
                                                  (300, 1000, 4, 40), (512, 4096, 3, 128),
                                                  (256, 4096, 8, 0), (1024, 11008, 3, 128)])
def test_device_rtn_quantizer_bit_exact(rows, cols, bits, group):
    # the oracle's quantize_rtn is pinned to the reference (test_oracle_golden.py)
    w = orc.gaussian(rows + cols + bits, rows, cols, 0.0, 0.02)
    words, sc, z = orc.quantize_rtn(w, bits, group)
    q = M.RtnQuantizer().quantize(torch.from_numpy(w), None, bits, group)
    assert np.array_equal(q.codes.words, words)
    assert np.array_equal(q.scales.view(np.uint32), np.asarray(sc, np.float32).view(np.uint32))
    assert np.array_equal(q.zeros.view(np.uint32), np.asarray(z, np.float32).view(np.uint32))
    # f32 weights = the reference on the widened values
    w32 = w.astype(np.float32)
    words32, sc32, z32 = orc.quantize_rtn(w32.astype(np.float64), bits, group)
    q32 = M.RtnQuantizer().quantize(torch.from_numpy(w32), None, bits, group)
    assert np.array_equal(q32.codes.words, words32)
    assert np.array_equal(q32.scales, np.asarray(sc32, np.float32))


@pytest.mark.gpu
def test_device_rtn_edge_grids():
    # flat groups (scale 1), signed zeros, ties at the extremes
    w = np.zeros((4, 16))
    w[1, 3] = -0.0
    w[1, 0] = 0.0
    w[2] = np.linspace(-1, 1, 16)
    w[3, ::2] = 0.5
    w[3, 1::2] = -0.5
    words, sc, z = orc.quantize_rtn(w, 4, 8)
    q = M.RtnQuantizer().quantize(torch.from_numpy(w), None, 4, 8)
    assert np.array_equal(q.codes.words, words)
    assert np.array_equal(q.scales.view(np.uint32), np.asarray(sc, np.float32).view(np.uint32))
    assert np.array_equal(q.zeros.view(np.uint32), np.asarray(z, np.float32).view(np.uint32))
    with pytest.raises(MlraError) as e:
        M.RtnQuantizer().quantize(torch.from_numpy(w), None, 5, 8)
    assert e.value.kind == "ConfigError"
    with pytest.raises(MlraError) as e:
        M.RtnQuantizer().quantize(torch.from_numpy(w), None, 4, 5)
    assert e.value.kind == "ConfigError"


@pytest.mark.gpu
def test_cb2_materialize_non_bf16_codebook():
    # magnitudes that are not bf16-exact take the f32 codebook layout
    rng = np.random.default_rng(9)
    cb = (rng.random((256, 8)) * 3.0 + 0.1).astype(np.float32)
    m = _random_cb2(130, 512, 64, seed=4)
    m = M.Cb2Matrix(m.rows, m.cols, m.group_size, m.codes, cb, m.scales)
    dq = M.Codebook2Quantizer(cb).upload(m)
    want = orc.cb2_dequantize_f32(m.codes, m.rows, m.cols, m.group_size, cb, m.scales)
    got = M.dequantize(dq, torch.float32).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    got16 = M.dequantize(dq, torch.bfloat16).view(torch.int16).cpu().numpy().view(np.uint16)
    assert np.array_equal(got16, orc.f32_to_bf16_bits(want))


@pytest.mark.gpu
@pytest.mark.parametrize("d_out,d_in,group,m", [(1024, 2048, 128, 700), (512, 768, 64, 1100)])
def test_cb2_fused_decode_matches_materialized(d_out, d_in, group, m, monkeypatch):
    # the fused path (codes decoded into the GEMM's smem tiles, Ŵ never in HBM)
    # feeds the tensor cores exactly the bf16 operands the hook materializes:
    # same MMA sequence -> bit-identical outputs; and nothing is charged to HBM
    monkeypatch.setenv("MLRA_GEMM", "2")
    w = orc.gaussian(31 + d_out, d_out, d_in, 0.0, 0.02)
    qz = M.Codebook2Quantizer()
    dq = qz.upload(qz.quantize(w, None, 2, group))
    x = to_bf16_dev(orc.bf16_round(orc.gaussian(32, m, d_in)))
    g = to_bf16_dev(orc.bf16_round(orc.gaussian(33, m, d_out)))
    fused = M.LpLinearContext(dq, S.RowMaterialize)
    assert fused.ledger_bytes() == 0
    y_f = M.lp_forward(fused, x, torch.float32)
    dx_f = M.lp_backward(fused, g, torch.float32)
    wctx = M.LpLinearContext(dq, S.WeightMaterialize)
    assert torch.equal(y_f, M.lp_forward(wctx, x, torch.float32))
    assert torch.equal(dx_f, M.lp_backward(wctx, g, torch.float32))
    monkeypatch.setenv("MLRA_CB2_HOOK", "1")  # the slabbed hook path, same numbers
    assert torch.equal(y_f, M.lp_forward(fused, x, torch.float32))
    wb = _deq_bf16(dq)
    assert rel_fro(f64(y_f), orc.bf16_round(orc.gaussian(32, m, d_in)) @ wb.T) < 1e-5
