"""The built-in "lut" Quantizer plugin (non-uniform levels, NF4 by default;
include/mlra.h mlra_lut_create): Ŵ = RN_f32(s · levels[c]) over the
reference's b-bit bitstream.

CPU tests pin the decode law (oracle/mlra_oracle.c orc_lut_dequant_f32) with
hand-computed known answers and a numpy restatement, the host packer against
the oracle's reference-pinned bitstream, and the quantizer's nearest-level
search. GPU tests check materialize() bit-exactly against the oracle, that the
fused GEMM (table decoded in the dequant warps, Ŵ never in HBM) produces
outputs bit-identical to the WeightMaterialize path, and a full layer against
the f64 oracle.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2309_16119_b200 import MlraError
from paper_2309_16119_b200 import modulora as M
from tests.conftest import rel_fro
from tests.gpu_util import f64, to_bf16_dev

S = M.MaterializationStrategy


def _random_lut(rows, cols, bits, group, seed, levels=None):
    rng = np.random.default_rng(seed)
    codes = rng.integers(0, 1 << bits, size=rows * cols, dtype=np.uint32)
    lv = M.normal_float_levels(bits) if levels is None else np.asarray(levels, np.float32)
    scales = (0.01 * (0.5 + rng.random((rows, cols // group)))).astype(np.float32)
    return M.LutMatrix(rows, cols, bits, group, M.PackedCodes(bits, rows * cols, M.pack_codes(codes, bits)),
                       lv, scales), codes


def _np_lut(codes, rows, cols, group, lv, scales):
    s = np.repeat(scales.reshape(rows, cols // group), group, axis=1)
    return (s * lv[codes.reshape(rows, cols)]).astype(np.float32)  # f32 * f32: one rounding


# ----------------------------------------------------------------------------- CPU
def test_lut_known_answer():
    lv = np.array([-1.0, -0.25, 0.5, 3.0], np.float32)
    codes = np.array([0, 1, 2, 3, 3, 2, 1, 0] * 2, np.uint32)  # 2 rows x 8, group 8
    words = orc.pack(codes, 2)
    got = orc.lut_dequantize_f32(words, 2, 8, 2, 8, lv, np.array([2.0, 0.5], np.float32))
    want = np.array([[-2.0, -0.5, 1.0, 6.0, 6.0, 1.0, -0.5, -2.0],
                     [-0.5, -0.125, 0.25, 1.5, 1.5, 0.25, -0.125, -0.5]], np.float32)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("bits,group", [(2, 8), (3, 16), (4, 64)])
def test_lut_oracle_matches_numpy(bits, group):
    m, codes = _random_lut(9, 128, bits, group, 3 + bits)
    got = orc.lut_dequantize_f32(m.codes.words, m.rows, m.cols, bits, group, m.levels, m.scales)
    assert np.array_equal(got.view(np.uint32), _np_lut(codes, 9, 128, group, m.levels, m.scales).view(np.uint32))


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
@pytest.mark.parametrize("n", [1, 5, 31, 32, 33, 100, 4099])
def test_pack_codes_matches_reference_bitstream(bits, n):
    c = np.random.default_rng(n * bits).integers(0, 1 << bits, n).astype(np.uint32)
    assert np.array_equal(M.pack_codes(c, bits), orc.pack(c, bits))
    assert np.array_equal(orc.unpack(M.pack_codes(c, bits), n, bits), c)


def test_pack_codes_rejects_out_of_range():
    with pytest.raises(MlraError):
        M.pack_codes(np.array([4], np.uint32), 2)


def test_normal_float_levels():
    for b in (2, 3, 4):
        lv = M.normal_float_levels(b)
        assert lv.size == 1 << b and np.all(np.diff(lv) > 0)
        assert lv[0] == -1.0 and lv[-1] == 1.0 and 0.0 in lv
    assert np.array_equal(M.normal_float_levels(4), M.NF4_LEVELS)
    with pytest.raises(MlraError):
        M.normal_float_levels(8)


@pytest.mark.parametrize("bits", [2, 3, 4])
def test_lut_quantizer_nearest_level(bits):
    w = orc.gaussian(40 + bits, 16, 256, 0.0, 0.02)
    q = M.LutQuantizer()
    m = q.quantize(w, None, bits, 64)
    codes = orc.unpack(m.codes.words, m.rows * m.cols, bits)
    x = w / np.repeat(m.scales.astype(np.float64), 64, axis=1)
    d = np.abs(x.reshape(-1, 1) - m.levels.astype(np.float64)[None, :])
    assert np.all(d[np.arange(codes.size), codes] <= d.min(1) + 1e-15)
    # absmax scaling: every group reaches a +-1 level
    assert np.allclose(np.abs(x).reshape(16, 4, 64).max(-1), 1.0)
    deq = orc.lut_dequantize_f32(m.codes.words, 16, 256, bits, 64, m.levels, m.scales)
    err = np.linalg.norm(deq - w) / np.linalg.norm(w)
    assert err < {2: 0.6, 3: 0.25, 4: 0.12}[bits]


def test_lut_quantizer_argument_errors():
    q = M.LutQuantizer()
    with pytest.raises(MlraError):
        q.quantize(np.zeros((4, 24)), None, 4, 12)
    with pytest.raises(MlraError):
        M.LutQuantizer(np.arange(8, dtype=np.float32)).quantize(np.zeros((4, 64)), None, 4, 64)
    m = q.quantize(np.zeros((2, 64)), None, 4, 32)  # all-zero groups: scale 1, code of level 0
    assert np.all(m.scales == 1.0)
    assert np.all(orc.lut_dequantize_f32(m.codes.words, 2, 64, 4, 32, m.levels, m.scales) == 0.0)


# ----------------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,bits,group", [
    (256, 512, 4, 64), (300, 264, 4, 8), (129, 384, 3, 128), (64, 1024, 2, 32),
    (17, 96, 3, 48), (512, 768, 4, 256)])
def test_lut_materialize_bit_exact(rows, cols, bits, group):
    m, _ = _random_lut(rows, cols, bits, group, rows + cols)
    dq = M.LutQuantizer().upload(m)
    info = dq.info()
    assert info["bits"] == bits and info["uncertified_groups"] == 0
    want = orc.lut_dequantize_f32(m.codes.words, rows, cols, bits, group, m.levels, m.scales)
    got = M.dequantize(dq, torch.float32).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    got16 = M.dequantize(dq, torch.bfloat16).view(torch.int16).cpu().numpy().view(np.uint16)
    assert np.array_equal(got16, orc.f32_to_bf16_bits(want))
    # a tile at an 8-aligned column offset, into a wider buffer
    t = M.dequantize_tile(dq, rows // 3, rows - rows // 3, 8, cols - 16, torch.float32).cpu().numpy()
    assert np.array_equal(t, want[rows // 3:, 8:cols - 8])


@pytest.mark.gpu
def test_lut_validation_errors():
    m, _ = _random_lut(8, 64, 4, 32, 1)
    q = M.LutQuantizer()
    bad = M.LutMatrix(8, 64, 8, 32, m.codes, np.zeros(256, np.float32), m.scales)
    with pytest.raises(MlraError) as e:
        q.upload(bad)
    assert e.value.status == 3
    lv = m.levels.copy()
    lv[3] = np.nan
    with pytest.raises(MlraError) as e:
        q.upload(M.LutMatrix(8, 64, 4, 32, m.codes, lv, m.scales))
    assert e.value.status == 6
    sc = m.scales.copy()
    sc[2, 1] = 0.0
    with pytest.raises(MlraError) as e:
        q.upload(M.LutMatrix(8, 64, 4, 32, m.codes, m.levels, sc))
    assert e.value.status == 6
    short = M.PackedCodes(4, 8 * 64, m.codes.words[:-1])
    with pytest.raises(MlraError) as e:
        q.upload(M.LutMatrix(8, 64, 4, 32, short, m.levels, m.scales))
    assert e.value.status == 7
    dq = q.upload(m)
    with pytest.raises(MlraError) as e:
        M.dequantize_tile(dq, 0, 8, 8, 12, torch.float32)
    assert e.value.status == 4


@pytest.mark.gpu
@pytest.mark.parametrize("d_out,d_in,bits,group,m", [
    (1024, 2048, 4, 64, 700), (512, 768, 3, 128, 1100), (768, 512, 2, 32, 96), (256, 1280, 4, 256, 4096)])
def test_lut_fused_decode_matches_weight_materialize(d_out, d_in, bits, group, m):
    # the fused path decodes the table into the GEMM's smem tiles: the tensor
    # cores see exactly the bf16 operands materialize() writes -> same MMA
    # sequence, bit-identical outputs; nothing is charged to HBM
    w = orc.gaussian(51 + d_out, d_out, d_in, 0.0, 0.02)
    qz = M.LutQuantizer()
    dq = qz.upload(qz.quantize(w, None, bits, group))
    x = to_bf16_dev(orc.bf16_round(orc.gaussian(52, m, d_in)))
    g = to_bf16_dev(orc.bf16_round(orc.gaussian(53, m, d_out)))
    wctx = M.LpLinearContext(dq, S.WeightMaterialize)
    y_w = M.lp_forward(wctx, x, torch.float32)
    dx_w = M.lp_backward(wctx, g, torch.float32)
    for strategy in (S.RowMaterialize, S.QuantizerMatvec):
        ctx = M.LpLinearContext(dq, strategy)
        assert ctx.ledger_bytes() == 0
        assert torch.equal(M.lp_forward(ctx, x, torch.float32), y_w)
        assert torch.equal(M.lp_backward(ctx, g, torch.float32), dx_w)
    wb = orc.bf16_round(M.dequantize(dq, torch.float32).cpu().numpy().astype(np.float64))
    assert rel_fro(f64(y_w), f64(x) @ wb.T) < 1e-5
    assert rel_fro(f64(dx_w), f64(g) @ wb) < 1e-5


@pytest.mark.gpu
def test_lut_off_ring_group_goes_through_hbm():
    # group 48 does not tile the Q ring: every strategy materializes Ŵ (ledger
    # says so) and the numbers still match the oracle
    d_out, d_in, m = 256, 384, 300
    qz = M.LutQuantizer()
    dq = qz.upload(qz.quantize(orc.gaussian(61, d_out, d_in, 0.0, 0.02), None, 4, 48))
    ctx = M.LpLinearContext(dq, S.RowMaterialize)
    assert ctx.ledger_bytes() == d_out * d_in * 2
    x = orc.bf16_round(orc.gaussian(62, m, d_in))
    wb = orc.bf16_round(M.dequantize(dq, torch.float32).cpu().numpy().astype(np.float64))
    y = f64(M.lp_forward(ctx, to_bf16_dev(x), torch.float32))
    assert rel_fro(y, x @ wb.T) < 1e-5


@pytest.mark.gpu
def test_lut_layer_forward_backward():
    d_out, d_in, m, r, alpha = 1024, 2048, 512, 16, 32.0
    w = orc.gaussian(71, d_out, d_in, 0.0, 0.02)
    qz = M.LutQuantizer()
    dq = qz.upload(qz.quantize(w, None, 4, 64))
    wb = orc.bf16_round(M.dequantize(dq, torch.float32).cpu().numpy().astype(np.float64))
    a = orc.gaussian(72, d_out, r, 0.0, 0.5).astype(np.float32)
    b = orc.gaussian(73, d_in, r, 0.0, 0.02).astype(np.float32)
    x = orc.bf16_round(orc.gaussian(74, m, d_in))
    g = orc.bf16_round(orc.gaussian(75, m, d_out))
    layer = M.ModuLoraLayer("nf4", dq, M.LoraAdapter(torch.from_numpy(a).cuda(),
                                                      torch.from_numpy(b).cuda(), r, alpha),
                            strategy=S.RowMaterialize)
    y, xb = M.layer_forward(layer, to_bf16_dev(x), out_dtype=torch.float32)
    dx = M.layer_backward(layer, to_bf16_dev(x), xb, to_bf16_dev(g), dx_dtype=torch.float32)
    yr, xbr = orc.layer_forward(wb, a, b, alpha, None, x)
    dxr, dar, dbr, _ = orc.layer_backward(wb, a, b, alpha, x, xbr, g)
    da, db = M.grads_of_adapter(layer)
    assert rel_fro(f64(y), yr) < 4e-3 and rel_fro(f64(dx), dxr) < 4e-3
    assert rel_fro(f64(da), dar) < 1e-4 and rel_fro(f64(db), dbr) < 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("m", [0, 1, 17, 257])
def test_lut_fused_ragged_token_counts(m):
    # tiny / ragged token counts take the pair kernel too (the table decode lives there)
    d_out, d_in = 512, 768
    qz = M.LutQuantizer()
    dq = qz.upload(qz.quantize(orc.gaussian(81, d_out, d_in, 0.0, 0.02), None, 4, 64))
    x = to_bf16_dev(orc.bf16_round(orc.gaussian(82, max(m, 1), d_in)))[:m]
    g = to_bf16_dev(orc.bf16_round(orc.gaussian(83, max(m, 1), d_out)))[:m]
    row = M.LpLinearContext(dq, S.RowMaterialize)
    wct = M.LpLinearContext(dq, S.WeightMaterialize)
    y = M.lp_forward(row, x, torch.float32)
    dx = M.lp_backward(row, g, torch.float32)
    assert y.shape == (m, d_out) and dx.shape == (m, d_in)
    assert torch.equal(y, M.lp_forward(wct, x, torch.float32))
    assert torch.equal(dx, M.lp_backward(wct, g, torch.float32))


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
def test_unpack_codes_inverts_pack(bits):
    c = np.random.default_rng(bits).integers(0, 1 << bits, 1001).astype(np.uint32)
    w = M.pack_codes(c, bits)
    assert np.array_equal(M.unpack_codes(w, c.size, bits), c)
    assert np.array_equal(M.unpack_codes(w, c.size, bits), orc.unpack(w, c.size, bits))
    with pytest.raises(MlraError):
        M.unpack_codes(w[:-1], c.size, bits)
