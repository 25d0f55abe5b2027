"""QuIP#-style path: the E8P lattice codebook
plugin "e8p" and the block randomized Hadamard transform (incoherence
processing).

The reference hosts such plugins but ships none, so the E8P
decode law is pinned by construction checks (every one of the 2^16 codes
decodes to a distinct point of E8's half-integer coset + 1/4), a hand-derived
known answer, and two independent restatements (oracle/mlra_oracle.c
orc_e8p_dequant_f32, modulora.e8p_decode) — then the device kernels
(materialize, the fused tile decode in the pair GEMM) are checked bit-exactly
against the oracle. The RHT is checked against an f64 numpy Walsh-Hadamard,
and the incoherent layer against the f64 layer on the un-rotated weights.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2309_16119_b200 import modulora as M
from tests.conftest import rel_fro
from tests.gpu_util import f64, to_bf16_dev


def _codes(rows, cols, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(0, 1 << 16, (rows, cols // 8), dtype=np.uint32).astype(np.uint16)


# ----------------------------------------------------------------------------- CPU
def test_e8p_abs_table_construction():
    t = orc.e8p_abs_table()  # 2|a|
    a, odd = M.e8p_abs_table()
    assert np.array_equal(a * 2, t) and t.shape == (256, 8)
    n4 = (t.astype(np.int64) ** 2).sum(1)  # 4|a|^2
    assert np.all(n4[:227] <= 40) and np.all(n4[227:] == 48)
    assert len({tuple(r) for r in t}) == 256 and set(np.unique(t)) <= {1, 3, 5}
    assert np.array_equal(odd, (t.sum(1) // 2) % 2 == 1)


def test_e8p_codes_are_distinct_lattice_points():
    codes = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    cw = M.e8p_decode(codes)
    assert len(np.unique(cw, axis=0)) == 1 << 16
    shift = np.where((codes.astype(np.uint32) >> 15) & 1, 0.25, -0.25)
    z = cw - shift[:, None]
    two = np.round(2 * z).astype(np.int64)
    assert np.allclose(2 * z, two) and np.all(two % 2 == 1)  # half-integers
    assert np.all((two.sum(1) // 2) % 2 == 0)                 # even sum: E8 = D8 u (D8 + 1/2)
    assert np.all((z ** 2).sum(1) <= 12.0 + 1e-12)


def test_e8p_known_answer():
    # pattern 1 = (1/2,...,1/2,3/2): sum 5 (odd); signs on entries 0 and 2; shift +1/4
    code = 1 | (1 << 8) | (1 << 10) | (1 << 15)
    # 2 negations among 0-6, odd sum -> entry 7 negated too (3 negations, odd total)
    want = np.array([-0.5, 0.5, -0.5, 0.5, 0.5, 0.5, 0.5, -1.5]) + 0.25
    assert np.array_equal(M.e8p_decode(np.array([code], np.uint16))[0], want)
    got = orc.e8p_dequantize_f32(np.array([[code]], np.uint16), 1, 8, 8, np.array([[2.0]], np.float32))
    assert np.array_equal(got[0], (2.0 * want).astype(np.float32))


def test_e8p_oracle_matches_python_restatement():
    rows, cols, g = 6, 64, 16
    codes = _codes(rows, cols, 3)
    sc = (0.01 * (0.5 + np.random.default_rng(4).random((rows, cols // g)))).astype(np.float32)
    got = orc.e8p_dequantize_f32(codes, rows, cols, g, sc)
    cw = M.e8p_decode(codes.ravel()).reshape(rows, cols)
    want = (np.repeat(sc, g, 1).astype(np.float32) * cw.astype(np.float32)).astype(np.float32)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_e8p_quantizer_beats_rtn_2bit():
    """The lattice codebook's point: lower MSE than scalar 2-bit RTN on
    Gaussian (post-incoherence) weights at the same 2 bits per weight."""
    w = orc.gaussian(17, 64, 512, 0.0, 1.0)
    m = M.E8pQuantizer().quantize(w, None, 2, 128)
    deq = orc.e8p_dequantize_f32(m.codes, 64, 512, 128, m.scales).astype(np.float64)
    words, sc, z = orc.quantize_rtn(w, 2, 128)
    rtn = orc.dequantize(words, 64, 512, 2, 128, sc, z)
    e_e8p = np.mean((deq - w) ** 2)
    e_rtn = np.mean((rtn - w) ** 2)
    assert e_e8p < 0.75 * e_rtn, (e_e8p, e_rtn)
    # nearest-point search: no single code change lowers a group's error
    v = w[0, :8] / m.scales[0, 0]
    best = M.e8p_decode(np.array([m.codes[0, 0]], np.uint16))[0]
    allc = M.e8p_decode(np.arange(1 << 16, dtype=np.uint32).astype(np.uint16))
    assert ((best - v) ** 2).sum() <= ((allc - v) ** 2).sum(1).min() + 1e-12


def _np_rht(x, signs, block, inverse=False):
    n = block
    h = np.array([[1.0]])
    while h.shape[0] < n:
        h = np.block([[h, h], [h, -h]])
    h /= np.sqrt(n)
    x = x.reshape(x.shape[0], -1, n)
    if not inverse:
        return np.einsum("ij,rbj->rbi", h, x * signs.reshape(-1, n)).reshape(x.shape[0], -1)
    return (np.einsum("ij,rbj->rbi", h, x) * signs.reshape(-1, n)).reshape(x.shape[0], -1)


# ----------------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,g", [(256, 512, 128), (6656, 17920, 128), (100, 72, 8)])
def test_e8p_materialize_bit_exact(rows, cols, g):
    codes = _codes(rows, cols, rows + cols)
    sc = (0.01 * (0.5 + np.random.default_rng(1).random((rows, cols // g)))).astype(np.float32)
    dq = M.E8pQuantizer().upload(M.E8pMatrix(rows, cols, g, codes, sc))
    want = orc.e8p_dequantize_f32(codes, rows, cols, g, sc)
    got = M.dequantize(dq, torch.float32).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    got16 = M.dequantize(dq, torch.bfloat16).view(torch.int16).cpu().numpy().view(np.uint16)
    assert np.array_equal(got16, orc.f32_to_bf16_bits(want))


@pytest.mark.gpu
def test_e8p_fused_decode_matches_hook_and_oracle():
    """RowMaterialize decodes E8P inside the pair GEMM (Q ring, Ŵ never in HBM,
    ledger 0); WeightMaterialize goes through the hook's whole-matrix
    materialize. Same bf16 operands, same MMA order -> bit-identical."""
    rows, cols, g, m, r = 512, 1024, 128, 700, 16
    codes = _codes(rows, cols, 9)
    sc = (0.02 * (0.5 + np.random.default_rng(2).random((rows, cols // g)))).astype(np.float32)
    dq = M.E8pQuantizer().upload(M.E8pMatrix(rows, cols, g, codes, sc))
    assert M.LpLinearContext(dq, M.MaterializationStrategy.RowMaterialize).ledger_bytes() == 0
    a32 = (0.02 * np.random.default_rng(3).standard_normal((rows, r))).astype(np.float32)
    b32 = (0.02 * np.random.default_rng(4).standard_normal((cols, r))).astype(np.float32)
    x64 = orc.bf16_round(orc.gaussian(5, m, cols))
    g64 = orc.bf16_round(orc.gaussian(6, m, rows))
    res = {}
    for strat in (M.MaterializationStrategy.RowMaterialize, M.MaterializationStrategy.WeightMaterialize):
        L = M.ModuLoraLayer("e8p", dq, M.LoraAdapter(torch.from_numpy(a32).cuda(),
                                                     torch.from_numpy(b32).cuda(), r, 32.0),
                            strategy=strat)
        y, xb = M.layer_forward(L, to_bf16_dev(x64), out_dtype=torch.float32)
        dx = M.layer_backward(L, to_bf16_dev(x64), xb, to_bf16_dev(g64), dx_dtype=torch.float32)
        res[strat] = (f64(y), f64(dx))
    r0, r1 = res.values()
    assert np.array_equal(r0[0], r1[0]) and np.array_equal(r0[1], r1[1])
    wbf = orc.bf16_round(orc.e8p_dequantize_f32(codes, rows, cols, g, sc))
    s = 32.0 / r
    A, B = a32.astype(np.float64), b32.astype(np.float64)
    y_ref = x64 @ wbf.T + orc.bf16_round(s * x64 @ B) @ orc.bf16_round(A).T
    dx_ref = g64 @ wbf + orc.bf16_round(s * g64 @ A) @ orc.bf16_round(B).T
    assert rel_fro(r0[0], y_ref) <= 1e-4 and rel_fro(r0[1], dx_ref) <= 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("block", [64, 512, 1024])
def test_rht_matches_f64_and_inverts(block):
    m, d = 33, 4 * block
    x64 = orc.bf16_round(orc.gaussian(block, m, d))
    s = M.random_signs(d, 7)
    y = M.rht(to_bf16_dev(x64), s, block, out_dtype=torch.float32)
    want = _np_rht(x64, s.cpu().numpy().astype(np.float64), block)
    assert rel_fro(f64(y), want) <= 1e-6
    back = M.rht(y.to(torch.bfloat16), s, block, inverse=True, out_dtype=torch.float32)
    assert rel_fro(f64(back), x64) <= 4e-3  # one bf16 rounding of the rotated values
    yi = M.rht(to_bf16_dev(x64), s, block, inverse=True, out_dtype=torch.float32)
    assert rel_fro(f64(yi), _np_rht(x64, s.cpu().numpy().astype(np.float64), block, True)) <= 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("block", [256, 512])
def test_rht_strided_rows_take_the_register_path(block):
    """Rows whose stride is not a 16-B multiple cannot feed the cp.async ring: the
    tensor-core RHT falls back to register prefetch — same values as the ring
    path on a contiguous copy (bit for bit) and as the f64 transform."""
    m, d = 37, 4 * block
    x64 = orc.bf16_round(orc.gaussian(block + 1, m, d))
    wide = torch.zeros(m, d + 2, dtype=torch.bfloat16, device="cuda")
    wide[:, :d] = to_bf16_dev(x64)
    strided = wide[:, :d]  # row stride d + 2 elements: 4-B but not 16-B aligned rows
    s = M.random_signs(d, 11)
    for inv in (False, True):
        y_str = M.rht(strided, s, block, inverse=inv, out_dtype=torch.float32)
        y_con = M.rht(strided.contiguous(), s, block, inverse=inv, out_dtype=torch.float32)
        assert torch.equal(y_str, y_con)
        want = _np_rht(x64, s.cpu().numpy().astype(np.float64), block, inv)
        assert rel_fro(f64(y_str), want) <= 1e-6


@pytest.mark.gpu
def test_incoherent_e8p_layer_is_the_unrotated_linear():
    """y = U^T(W~ V x) + s(xB)A^T + bias with W~ quantized by E8P in the rotated
    basis equals the layer on W = U^T W~ V (exactly, in f64) with A = U^T A~,
    B = V^T B~; checked against that f64 layer at the bf16 bar."""
    d_out, d_in, g, m, r, blk = 512, 1024, 128, 300, 8, 512
    w = orc.gaussian(31, d_out, d_in, 0.0, 0.02)
    u, v = M.random_signs(d_out, 1), M.random_signs(d_in, 2)
    un, vn = u.cpu().numpy().astype(np.float64), v.cpu().numpy().astype(np.float64)
    # W~ = U W V^T  (U = H diag(u) blockwise): rotate rows then columns
    wt = _np_rht(_np_rht(w.T, un, blk).T.copy(), vn, blk)
    qm = M.E8pQuantizer().quantize(wt, None, 2, g)
    dq = M.E8pQuantizer().upload(qm)
    a_t = (0.02 * np.random.default_rng(5).standard_normal((d_out, r))).astype(np.float32)
    b_t = (0.02 * np.random.default_rng(6).standard_normal((d_in, r))).astype(np.float32)
    bias = (0.1 * np.random.default_rng(7).standard_normal(d_out)).astype(np.float32)
    bias_t = M.IncoherentLayer.rotated_bias(torch.from_numpy(bias).cuda(), u, blk)
    inner = M.ModuLoraLayer("inc", dq, M.LoraAdapter(torch.from_numpy(a_t).cuda(),
                                                     torch.from_numpy(b_t).cuda(), r, 16.0),
                            bias=bias_t)
    layer = M.IncoherentLayer(inner, u, v, blk)
    x64 = orc.bf16_round(orc.gaussian(8, m, d_in))
    g64 = orc.bf16_round(orc.gaussian(9, m, d_out))
    y, saved = layer.forward(to_bf16_dev(x64))
    dx = layer.backward(saved, to_bf16_dev(g64))
    # the equivalent un-rotated layer in f64
    wq = orc.e8p_dequantize_f32(qm.codes, d_out, d_in, g, qm.scales).astype(np.float64)
    w_eq = _np_rht(_np_rht(wq, vn, blk, inverse=True).T.copy(), un, blk, inverse=True).T  # U^T W~ V
    A = _np_rht(a_t.astype(np.float64).T.copy(), un, blk, inverse=True).T   # U^T A~
    B = _np_rht(b_t.astype(np.float64).T.copy(), vn, blk, inverse=True).T   # V^T B~
    s = 16.0 / r
    y_ref = x64 @ w_eq.T + s * (x64 @ B) @ A.T + bias.astype(np.float64)
    dx_ref = g64 @ w_eq + s * (g64 @ A) @ B.T
    # bf16 at each transform boundary (V x, W~ operands, the U^T input, the output)
    assert rel_fro(f64(y), y_ref) <= 1.2e-2
    assert rel_fro(f64(dx), dx_ref) <= 1.2e-2
    da, db = M.grads_of_adapter(inner)  # gradients of A~, B~ (the rotated-basis adapters)
    xt = _np_rht(x64, vn, blk)
    gt = _np_rht(g64, un, blk)
    assert rel_fro(f64(da), s * gt.T @ (xt @ b_t.astype(np.float64))) <= 2e-2
    assert rel_fro(f64(db), s * xt.T @ (gt @ a_t.astype(np.float64))) <= 2e-2
